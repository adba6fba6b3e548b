#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
for wf in estimate; do
timeout 900 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --workflow $wf > gpurun_out/bench_$wf.json 2> gpurun_out/bench_$wf.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$wf.json')); print('$wf', round(d['ms_per_step'],2), d['config']['stage_ms'], d['config'].get('estimation_share'), d['roofline']['kernel_ms_per_step'])"; tail -2 gpurun_out/bench_$wf.err
done
timeout 1200 ncu --set full --clock-control none --import-source on -k k_hash_block -c 1 -s ${KSKIP:-6} -o gpurun_out/it_prof -f python tools/run_once.py rmat20 > gpurun_out/it_ncu.log 2>&1; tail -1 gpurun_out/it_ncu.log
