mkdir -p gpurun_out
for lib in paper_1909_04153_b200/lib/libbsq.so "$@"; do
  BSQ_LIB=$lib python tools/ab_kernels.py --steps 20 --precision fp32 2>&1 | tail -1
done > gpurun_out/ab32.log
cat gpurun_out/ab32.log
