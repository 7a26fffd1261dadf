# ncu capture of the fp32 stage kernel (one AB3 step of the bench workload)
mkdir -p gpurun_out
python tools/profile_step.py --steps 1 --precision fp32 > gpurun_out/p32_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_stage -s 3 -c 1 -o gpurun_out/p32_stage -f \
  python tools/profile_step.py --steps 1 --precision fp32 > gpurun_out/p32_ncu.log 2>&1
tail -2 gpurun_out/p32_ncu.log
