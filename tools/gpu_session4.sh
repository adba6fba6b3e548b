#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --maxfail=10 -p no:cacheprovider -x > gpurun_out/pytest_gpu.txt 2>&1
tail -15 gpurun_out/pytest_gpu.txt
for c in rmat16 poisson64 rect; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  tail -2 gpurun_out/bench_$c.err
done
timeout 1500 python bench.py --config rmat20 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_rmat20.json 2> gpurun_out/bench_rmat20.err
tail -3 gpurun_out/bench_rmat20.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rmat18.csv python tools/run_once.py rmat18 > gpurun_out/ncu_b.log 2>&1
