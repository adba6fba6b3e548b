#!/bin/bash
mkdir -p gpurun_out
H=$PWD/paper_2604_19004_b200/libsgb200_half.so
SGB200_LIB=$H timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_half.txt 2>&1; tail -3 gpurun_out/pytest_half.txt
for lib in libsgb200.so libsgb200_half.so; do
SGB200_LIB=$PWD/paper_2604_19004_b200/$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_rmat20_$lib.json 2> gpurun_out/bench_rmat20_$lib.err
python -c "import json,sys; d=json.loads(open('gpurun_out/bench_rmat20_$lib.json').read()); print('$lib', d['value'], d['ms_per_step'], d['config']['stage_ms'], d['roofline']['kernel_ms_per_step'])"
tail -2 gpurun_out/bench_rmat20_$lib.err
done
