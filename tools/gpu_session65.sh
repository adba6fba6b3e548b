#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 2 > gpurun_out/bench_rmat20.json 2> gpurun_out/bench_rmat20.err
python -c "import json,sys; d=json.loads(open('gpurun_out/bench_rmat20.json').read()); print(d['value'], d['ms_per_step'], d['e2e'], d['clocks'])"
tail -3 gpurun_out/bench_rmat20.err
