"""A/B builds: relink libbsq.so with some sources recompiled under extra -D
flags, into paper_1909_04153_b200/lib/variants/<name>.so.  Load one with
BSQ_LIB=<path> (paper_1909_04153_b200/_native.py honours it for A/B runs).

    python tools/build_variant.py <name> <source.cu>[,<source.cu>] [-DFOO ...]

(both precision objects of each named source are rebuilt with the extra flags)
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
objs, todo = [], []
for src, obj, prec in B.jobs():
    if src in srcs:
        obj = os.path.join(vdir, os.path.basename(obj))
        todo.append((src, obj, prec))
    objs.append(obj)
for log in B.compile_jobs(todo, extra=defs):
    for ln in log.splitlines():
        if "registers" in ln or "spill" in ln or ln.endswith("]"):
            print(ln.strip())
out = os.path.join(B.OUT_DIR, "variants", name + ".so")
B.link(objs, out)
print(out)
