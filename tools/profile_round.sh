#!/bin/bash
# One GPU call: bench (plain), then the ncu launch list and a --set full
# capture of one AB3 step of the bench workload.  Outputs in gpurun_out/$TAG*.
#   gpurun --timeout 1500 -- 'bash tools/profile_round.sh r1c'
set -u
TAG=${1:-prof}
OUT=gpurun_out
mkdir -p $OUT
python bench.py --steps 20 --warmup 3 > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench rc=$?"
python tools/profile_step.py --steps 2 > $OUT/${TAG}_plain.log 2>&1
echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv python tools/profile_step.py --steps 2 \
    > $OUT/${TAG}_ncu_l.log 2>&1
echo "launch list rc=$?"
# one AB3 step with speculation: skip the initial extrema, step 1 (ghost_t,
# stage, ghost_n, solve1, correct, solve2, final + the queued ghost_t (with the
# frame save) and stage = 9) and steps 2-3 (7 each), then capture step 4's 7
# launches (ghost_n .. final, and the queued ghost_t, stage of step 5)
ncu --set full --clock-control none --import-source on -s 24 -c 7 \
    -o $OUT/${TAG} -f python tools/profile_step.py --steps 2 > $OUT/${TAG}_ncu.log 2>&1
echo "full rc=$?"
