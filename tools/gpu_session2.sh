#!/bin/bash
set -x
mkdir -p gpurun_out
for c in rmat16 poisson64 rect rmat20; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --cpu-seconds 8 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  tail -2 gpurun_out/bench_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rmat18.csv python bench.py --config rmat18 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_b.log 2>&1
