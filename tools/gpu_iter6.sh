#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -m gpu -q -x > gpurun_out/it_pytest.txt 2>&1; tail -2 gpurun_out/it_pytest.txt
for wf in auto estimate; do
timeout 900 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --workflow $wf > gpurun_out/bench_$wf.json 2> gpurun_out/bench_$wf.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$wf.json')); print('$wf', round(d['ms_per_step'],2), d['config']['stage_ms'], d['config'].get('estimation_share'), d['roofline']['kernel_ms_per_step'])"; tail -2 gpurun_out/bench_$wf.err
done
