"""Build experiment variants of libtoep_b200.so (compile-time macro sets) for A/B timing on one box.

    python tools/build_variants.py NAME=-DFOO=1,-DBAR=0 NAME2=...
    # then on the GPU: TOEP_LIB=paper_1502_03162_b200/build/variants/libtoep_NAME.so python bench.py ...
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1502_03162_b200 import _build  # noqa: E402

OUT = os.path.join(_build.BUILD, "variants")


def build_variant(name, defines):
    os.makedirs(os.path.join(OUT, name), exist_ok=True)
    objs = []
    procs = []
    for src in _build.SOURCES:
        o = os.path.join(OUT, name, src.replace(".cu", ".o"))
        objs.append(o)
        procs.append(subprocess.Popen([_build._nvcc(), *_build.NVCC_FLAGS, *defines, "-c",
                                       os.path.join(_build.CSRC, src), "-o", o]))
    for p in procs:
        if p.wait():
            raise SystemExit("nvcc failed for " + name)
    lib = os.path.join(OUT, "libtoep_%s.so" % name)
    subprocess.check_call([_build._nvcc(), *_build.NVCC_FLAGS, "-shared", *objs, "-o", lib])
    shutil.rmtree(os.path.join(OUT, name))  # objects are not needed on the GPU box
    print(lib)


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        name, _, defs = arg.partition("=")
        build_variant(name, [d for d in defs.split(",") if d])
