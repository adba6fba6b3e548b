#!/bin/bash
SGB200_LIB=$PWD/paper_2604_19004_b200/libsgb200_prof.so timeout 600 python tools/phase_prof.py rmat20 2>&1 | tail -10
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/b.json 2> gpurun_out/b.err
python -c "import json,sys; d=json.loads(open('gpurun_out/b.json').read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_step'])"
