#!/bin/bash
# Config-5 sparse path: launch list (per-kernel share of an iteration) and one full ncu capture
# of the top kernel.  Outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -s 40 -c 60 --csv \
  --log-file gpurun_out/sparse_launches.csv python tools/sparse_bench.py 1000000 200000 6 > gpurun_out/sparse_ncu.log 2>&1
echo "sparse launch list rc=$?"
