mkdir -p gpurun_out
V=paper_1909_04153_b200/lib/variants
for lib in paper_1909_04153_b200/lib/libbsq.so $V/noprefetch.so $V/nodry.so $V/neither.so paper_1909_04153_b200/lib/libbsq.so; do
  BSQ_LIB=$lib python tools/ab_kernels.py --steps 20 2>&1 | tail -1
done > gpurun_out/ab1.log
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2 >> gpurun_out/ab1.log
cat gpurun_out/ab1.log
