#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -m gpu -x -q 2>&1 | tail -1
for c in rect poisson64; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$c.json').read()); print('$c', d['value'], d['ms_per_step'], d['config']['stage_ms'])"
done
