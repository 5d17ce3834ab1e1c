#!/bin/bash
# Round-2 profile evidence for the re-sequenced single-read kernel (one GPU session): launch
# lists of config 4 (kkt=False loop and the default fit() with the KKT pass) and one full ncu
# capture of the pass and of the KKT pass.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
A="--steps 8 --warmup 3 --no-e2e --no-cpu"
timeout 300 python bench.py --config 4 $A > gpurun_out/plain_c4.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 150 --csv \
  --log-file gpurun_out/r02_launches_config4.csv python bench.py --config 4 $A > gpurun_out/ncu_c4.log 2>&1
echo "launch list config 4 rc=$?"
timeout 300 python tools/kkt_cost.py 1048576 > gpurun_out/plain_kkt.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 80 -c 100 --csv \
  --log-file gpurun_out/r02_launches_config4_kkt.csv python tools/kkt_cost.py 1048576 > gpurun_out/ncu_kkt.log 2>&1
echo "kkt launch list rc=$?"
timeout 300 python bench.py $A > gpurun_out/plain_full.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_pass_tc -s 3 -c 1 \
  -f -o gpurun_out/r02_prof_fused python bench.py $A > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
