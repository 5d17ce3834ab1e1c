#!/bin/bash
# One GPU session: the bench line of every BASELINE config and the reference arm -> gpurun_out/r02_bench_*.json
mkdir -p gpurun_out
python bench.py --steps 50 --warmup 5 > gpurun_out/r02_bench_config4.json 2> gpurun_out/r02_bench_config4.err; echo "config 4 rc=$?"
for c in 1 2 3; do
  timeout 600 python bench.py --config $c --steps 100 --warmup 10 > gpurun_out/r02_bench_config$c.json 2> gpurun_out/r02_bench_config$c.err; echo "config $c rc=$?"
done
timeout 900 python bench.py --config 5 --steps 32 --warmup 4 > gpurun_out/r02_bench_config5.json 2> gpurun_out/r02_bench_config5.err; echo "config 5 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_bench_reference_arm.err; echo "reference rc=$?"
for f in gpurun_out/r02_bench_*.json; do echo $f; tail -1 $f | cut -c1-260; done
