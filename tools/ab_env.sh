#!/bin/bash
# A/B of runtime switches (env assignments) on the shipped library, one GPU:
#   gpurun -- 'bash tools/ab_env.sh <tag> "BSQ_PDL=0" "BSQ_PDL=1"'
mkdir -p gpurun_out
TAG=${1:-abenv}; shift
for rep in 1 2; do
  for e in "$@"; do
    echo -n "$e "; env $e python tools/ab_kernels.py --steps 20 ${AB_ARGS:-} 2>&1 | tail -1
  done
done > gpurun_out/$TAG.log
cat gpurun_out/$TAG.log
