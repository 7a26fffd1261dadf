#!/bin/bash
# A/B per-kernel times of library variants (tools/build_variant.py), one GPU.
#   gpurun -- 'bash tools/ab_run.sh <tag> [variant names...]'
# Each library runs twice, interleaved (A B C A B C), to expose drift.
mkdir -p gpurun_out
TAG=${1:-ab}; shift
V=paper_1909_04153_b200/lib/variants
libs="paper_1909_04153_b200/lib/libbsq.so"
for n in "$@"; do libs="$libs $V/$n.so"; done
for rep in 1 2; do
  for lib in $libs; do
    BSQ_LIB=$lib python tools/ab_kernels.py --steps 20 ${AB_ARGS:-} 2>&1 | tail -1
  done
done > gpurun_out/$TAG.log
cat gpurun_out/$TAG.log
