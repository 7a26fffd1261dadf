#!/bin/bash
# One GPU call: ncu --set full capture of one fp32 AB3 step of the bench
# workload (same launch order as profile_round.sh).  Outputs in gpurun_out/$TAG*.
set -u
TAG=${1:-p32}
OUT=gpurun_out
mkdir -p $OUT
python tools/profile_step.py --steps 2 --precision fp32 > $OUT/${TAG}_plain.log 2>&1
echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -s 24 -c 7 \
    -o $OUT/${TAG} -f python tools/profile_step.py --steps 2 --precision fp32 > $OUT/${TAG}_ncu.log 2>&1
echo "full rc=$?"
