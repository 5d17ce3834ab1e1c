#!/bin/bash
# One GPU session: bench line of every dense BASELINE config (no e2e / cpu legs
# for the secondary configs) and the config-5 sparse timing.  Outputs under gpurun_out/.
mkdir -p gpurun_out
for c in 1 2 3; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  echo "config $c rc=$?"; tail -1 gpurun_out/bench_c$c.json | cut -c1-400
done
