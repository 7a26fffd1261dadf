# A/B per-kernel times of library variants (tools/build_variant.py), one GPU
mkdir -p gpurun_out
V=paper_1909_04153_b200/lib/variants
for lib in paper_1909_04153_b200/lib/libbsq.so "$@"; do
  BSQ_LIB=$lib python tools/ab_kernels.py --steps 20 2>&1 | tail -1
done > gpurun_out/ab.log
cat gpurun_out/ab.log
