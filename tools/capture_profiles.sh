#!/bin/bash
# One GPU session: bench line, clocks, ncu launch list of the same command,
# one full ncu capture of the fused pass.  Outputs under gpurun_out/.
set -u
ARGS="--steps 32 --warmup 3"
mkdir -p gpurun_out
timeout 600 python bench.py $ARGS > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
tail -1 gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 5 -c 120 --csv \
  --log-file gpurun_out/launches.csv python bench.py $ARGS --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_pass_tc -s 3 -c 1 \
  -o gpurun_out/prof_fused python bench.py $ARGS --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
