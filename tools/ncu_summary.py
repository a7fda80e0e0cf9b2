"""Condense an ncu report / launch list into a small text summary for profiles/.

    python tools/ncu_summary.py report.ncu-rep > profiles/<name>.txt
    python tools/ncu_summary.py --launches launches.csv > profiles/<name>_launches.txt
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print("ncu --set full report:", path)
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print("\nkernel:", d.get("Kernel Name"))
        for k in KEYS:
            if k in d:
                print("  %-62s %s %s" % (k, d[k], u.get(k, "")))
        st = [(k, float(v)) for k, v in d.items()
              if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active\.ratio$", k) and v]
        st.sort(key=lambda x: -x[1])
        print("  warp stall reasons (cycles per issued instruction):")
        for k, v in st[:8]:
            print("    %-40s %.3f" % (k.replace("smsp__average_warps_issue_stalled_", "").replace(
                "_per_issue_active.ratio", ""), v))
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    if len(rows) > 2:
        h = rows[1]
        data = []
        for r in rows[2:]:  # the first kernel's section (a report may hold several)
            if r and r[0] == "Kernel Name":
                break
            data.append(r)
        si, wi, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        tot = sum(float(r[wi] or 0) for r in data) or 1.0
        ex = sum(float(r[ei] or 0) for r in data) or 1.0
        cs, ce = collections.Counter(), collections.Counter()
        for r in data:
            t = r[si].split()
            if not t:
                continue
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            cs[op] += float(r[wi] or 0)
            ce[op] += float(r[ei] or 0)
        print("  (SASS source page, first kernel of the report)")
        print("  executed-instruction mix:", ", ".join("%s %.1f%%" % (k, 100 * v / ex) for k, v in ce.most_common(10)))
        print("  stall-sample share by opcode:", ", ".join("%s %.1f%%" % (k, 100 * v / tot) for k, v in cs.most_common(10)))


def launches(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[i], rows[i + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    unit = "ns"
    for r in data:
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        agg[r[ki][:90]].append(v)
    tot = sum(sum(v) for v in agg.values())
    print("ncu launch list (--metrics gpu__time_duration.sum, cold-cache, serialised):", path)
    print("%6s %14s %7s %14s  %s" % ("count", "total " + unit, "share", "avg " + unit, "kernel"))
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print("%6d %14.0f %6.1f%% %14.0f  %s" % (len(v), sum(v), 100 * sum(v) / tot, sum(v) / len(v), k))


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[1])
