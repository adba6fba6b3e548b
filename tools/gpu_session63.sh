#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "download or identity" 2>&1 | tail -2
python tools/d2h_bench.py 16 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_rmat20.json 2> gpurun_out/bench_rmat20.err
python -c "import json,sys; d=json.loads(open('gpurun_out/bench_rmat20.json').read()); print(d['value'], d['ms_per_step'], d['e2e'])"
tail -3 gpurun_out/bench_rmat20.err
