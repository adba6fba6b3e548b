#!/bin/bash
# parity subset + bench variants (env list in VARIANTS) + ncu of k_win
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -m gpu -q -x > gpurun_out/it_pytest.txt 2>&1; tail -2 gpurun_out/it_pytest.txt
for v in ${VARIANTS:-"X=1"}; do
env $v timeout 900 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; python -c "
import json; d=json.load(open('gpurun_out/it_bench.json')); print('$v', round(d['ms_per_step'],2), d['config']['stage_ms'], d['roofline']['kernel_ms_per_step'])"; tail -2 gpurun_out/it_bench.err
done
[ "${NCU:-1}" = "1" ] && timeout 1200 ncu --set full --clock-control none --import-source on -k ${KSEL:-k_win} -c 1 -o gpurun_out/it_prof -f python tools/run_once.py rmat20 > gpurun_out/it_ncu.log 2>&1; tail -1 gpurun_out/it_ncu.log
