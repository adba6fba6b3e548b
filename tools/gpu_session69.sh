#!/bin/bash
mkdir -p gpurun_out
L=$PWD/paper_2604_19004_b200
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_cols.txt 2>&1; tail -2 gpurun_out/pytest_cols.txt
for lib in libsgb200.so libsgb200_sepcols.so; do
SGB200_LIB=$L/$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_$lib.json 2> gpurun_out/b_$lib.err
python -c "import json,sys; d=json.loads(open('gpurun_out/b_$lib.json').read()); print('$lib', d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_step'].get('k_expand'), d['roofline']['kernel_ms_per_step']['k_bmr'])"
done
