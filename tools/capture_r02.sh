#!/bin/bash
# Round-2 profile evidence (one GPU session): launch lists of config 4 (default kkt=False loop and
# the default fit() with the fused KKT pass), configs 1-3, and one full ncu capture of the fused
# pass and of the KKT pass.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
A="--steps 8 --warmup 3 --no-e2e --no-cpu"
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c $A > gpurun_out/plain_c$c.log 2>&1 &&
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 150 --csv \
    --log-file gpurun_out/r02_launches_config$c.csv python bench.py --config $c $A > gpurun_out/ncu_c$c.log 2>&1
  echo "launch list config $c rc=$?"
done
timeout 300 python tools/kkt_cost.py 1048576 > gpurun_out/plain_kkt.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 80 -c 100 --csv \
  --log-file gpurun_out/r02_launches_config4_kkt.csv python tools/kkt_cost.py 1048576 > gpurun_out/ncu_kkt.log 2>&1
echo "kkt launch list rc=$?"
timeout 300 python bench.py $A > gpurun_out/plain_full.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_pass_tc -s 3 -c 1 \
  -f -o gpurun_out/r02_prof_fused python bench.py $A > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
