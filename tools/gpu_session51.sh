#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
for c in rect poisson64; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$c.json').read()); print('$c', d['value'], d['ms_per_step'], d['config']['stage_ms'], d['roofline']['kernel_ms_per_step'])"
tail -2 gpurun_out/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_rect.csv python tools/run_once.py rect > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/launches_rect.csv 6
