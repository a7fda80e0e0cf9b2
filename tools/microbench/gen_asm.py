"""Emit an inline-PTX tap loop with a warp-uniform jump table (brx.idx.uni).

Operands: %0..%R-1 accumulators (+f), %R..%R+NW-1 window registers (f),
then the tap pointer (l).  Each case o performs acc[r] += v * win[r + KW - o]
and then loads the next (offset, value) tap and dispatches on it; offset KW is
the end-of-list sentinel.
"""
import sys


def gen(R, KW, name):
    NW = R + KW
    p = R + NW
    lines = []
    a = lines.append
    a("{")
    a(".reg .u32 jo, jn;")
    a(".reg .f32 jv, jw;")
    a(".reg .u64 jp;")
    a(f"mov.u64 jp, %{p};")
    a("ld.global.nc.v2.u32 {jo, jn}, [jp];")
    a("mov.b32 jv, jn;")
    a("add.u64 jp, jp, 8;")
    targets = ", ".join([f"JC{o}" for o in range(KW)] + ["JEND"])
    a(f"JTBL: .branchtargets {targets};")
    a("brx.idx.uni jo, JTBL;")
    for o in range(KW):
        a(f"JC{o}:")
        a("ld.global.nc.v2.u32 {jo, jn}, [jp];")
        a("add.u64 jp, jp, 8;")
        for r in range(R):
            a(f"fma.rn.f32 %{r}, jv, %{R + r + KW - o}, %{r};")
        a("mov.b32 jv, jn;")
        a("brx.idx.uni jo, JTBL;")
    a("JEND:")
    a("}")
    body = "\\n\\t".join(lines)
    return f'#define {name} "{body}\\n"\n'


if __name__ == "__main__":
    out = []
    for R, KW in [(20, 100), (12, 100), (28, 100)]:
        out.append(gen(R, KW, f"JT_ASM_R{R}_K{KW}"))
    open(sys.argv[1], "w").write("".join(out))
