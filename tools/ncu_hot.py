"""Top SASS instructions by warp-stall samples from an ncu report (source page CSV).

    python tools/ncu_hot.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
i_src, i_s, i_ex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stall = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
num = lambda v: int(v) if v.isdigit() else 0
tot = sum(num(r[i_s]) for r in data)
print("total samples", tot)
for r in sorted(data, key=lambda r: -num(r[i_s]))[:n]:
    st = sorted(((num(r[i]), h[6:]) for i, h in stall), reverse=True)[:2]
    print(r[0][-5:], f"{100 * num(r[i_s]) / tot:5.1f}%", r[i_ex].rjust(10), r[i_src].strip()[:58].ljust(58),
          " ".join(f"{h}={v}" for v, h in st if v))
