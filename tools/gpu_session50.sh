#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_rmat20.json 2> gpurun_out/bench_rmat20.err
cat gpurun_out/bench_rmat20.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['roofline']))"
tail -3 gpurun_out/bench_rmat20.err
