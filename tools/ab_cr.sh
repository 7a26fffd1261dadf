for lib in paper_1909_04153_b200/lib/libbsq.so "$@"; do
  BSQ_LIB=$lib python tools/ab_kernels.py --solver cr --steps 10 2>&1 | tail -1
done
