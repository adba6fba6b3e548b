#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 1500 python bench.py --config rmat20 --steps 3 --warmup 3 --cpu-seconds 15 > gpurun_out/bench_rmat20.json 2> gpurun_out/bench_rmat20.err
tail -2 gpurun_out/bench_rmat20.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_rmat20.csv python tools/run_once.py rmat20 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_rmat20.csv 12
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_bmr -c 1 -o gpurun_out/prof_bmr_rmat20 python tools/run_once.py rmat20 > /dev/null 2>&1
ls -la gpurun_out/prof_bmr_rmat20.ncu-rep
