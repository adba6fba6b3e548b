#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rmat18.csv python tools/run_once.py rmat18 > gpurun_out/ncu_b.log 2>&1
python tools/ncu_summary.py gpurun_out/launches_rmat18.csv 8
timeout 1500 python bench.py --config rmat20 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_rmat20.json 2> gpurun_out/bench_rmat20.err
tail -2 gpurun_out/bench_rmat20.err
python -c "
import json; d=json.load(open('gpurun_out/bench_rmat20.json')); print('GF', round(d['value'],2), 'ms', round(d['ms_per_step'],3), d['config']['stage_ms'], 'e2e', d['e2e'])"
