"""A/B builds: relink libbsq.so with some sources recompiled under extra -D
flags, into paper_1909_04153_b200/lib/variants/<name>.so.  Load one with
BSQ_LIB=<path> (paper_1909_04153_b200/_native.py honours it for A/B runs).

    python tools/build_variant.py <name> <source.cu>[,<source.cu>] [-DFOO ...]
"""

import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_04153_b200 import build as B  # noqa: E402

name, srcs, defs = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
B.build()
vdir = os.path.join(B.OUT_DIR, "variants", name)
os.makedirs(vdir, exist_ok=True)
objs = []
for src in B.SOURCES:
    obj = os.path.join(B.OUT_DIR, os.path.splitext(src)[0] + ".o")
    if src in srcs:
        obj = os.path.join(vdir, os.path.splitext(src)[0] + ".o")
        cmd = [B.nvcc(), *B.FLAGS, *defs, "-c", os.path.join(B.SRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stdout + r.stderr)
        for ln in r.stderr.splitlines():
            if "registers" in ln or "spill" in ln:
                print(src, ln.strip())
    objs.append(obj)
out = os.path.join(B.OUT_DIR, "variants", name + ".so")
subprocess.run([B.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out,
                *objs, "-ccbin", "/usr/bin/g++", "-lcudart", "-lpthread"], check=True)
print(out)
