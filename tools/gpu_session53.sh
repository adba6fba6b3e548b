#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
for c in rect poisson64 rmat16; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$c.json').read()); print('$c', d['value'], d['ms_per_step'], d['config']['stage_ms'], d['roofline']['kernel_ms_per_step'], d['clocks'])"
tail -2 gpurun_out/bench_$c.err
done
python tools/timeline.py poisson64 2 > gpurun_out/tl_poisson.txt 2>&1; head -14 gpurun_out/tl_poisson.txt
