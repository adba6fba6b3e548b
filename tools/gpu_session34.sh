#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
SGB200_LIB=paper_2604_19004_b200/libsgb200_prof.so timeout 600 python tools/phase_prof.py rmat18 2>&1 | tail -10 | head -7
timeout 1500 python bench.py --config rmat20 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_rmat20.json 2> gpurun_out/bench_rmat20.err
tail -2 gpurun_out/bench_rmat20.err
python -c "
import json; d=json.load(open('gpurun_out/bench_rmat20.json')); print('GF', round(d['value'],2), 'ms', round(d['ms_per_step'],3), d['config']['stage_ms'])"
