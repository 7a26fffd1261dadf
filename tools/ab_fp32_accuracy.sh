# fp32 accuracy (eta rel-L2 vs the fp64 reference, tests/test_gpu_fp32.py) and
# step time of library variants: bash tools/ab_fp32_accuracy.sh <variant.so> ...
for lib in paper_1909_04153_b200/lib/libbsq.so "$@"; do
  echo "== $lib"
  BSQ_LIB=$lib python -m pytest tests/test_gpu_fp32.py -q -s 2>&1 | grep -E 'rel-L2|passed|failed' | sed 's/, dt.*//'
  BSQ_LIB=$lib python tools/ab_kernels.py --steps 20 --precision fp32 2>&1 | tail -1
done
