#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_rmat18.csv python tools/run_once.py rmat18 > gpurun_out/ncu_b.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_rect.csv python tools/run_once.py rect > gpurun_out/ncu_r.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_poisson.csv python tools/run_once.py poisson64 > gpurun_out/ncu_p.log 2>&1
timeout 1500 python bench.py --config rmat20 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_rmat20.json 2> gpurun_out/bench_rmat20.err
tail -3 gpurun_out/bench_rmat20.err
