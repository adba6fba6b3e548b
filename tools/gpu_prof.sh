#!/bin/bash
# One ncu --set full capture of a kernel on R-MAT-20 (KREGEX, KCOUNT), plus a short bench.
mkdir -p gpurun_out
[ "${BENCH:-1}" = "1" ] && timeout 900 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; python -c "
import json; d=json.load(open('gpurun_out/it_bench.json')); print(d['ms_per_step'], d['config']['stage_ms'], d['roofline']['kernel_ms_per_step'], d['roofline'].get('units_per_launch'))"; tail -3 gpurun_out/it_bench.err
timeout 1200 ncu --set full --clock-control none --import-source on -k ${KSEL:-k_win} -c ${KCOUNT:-1} -o gpurun_out/it_prof -f python tools/run_once.py ${CFG:-rmat20} > gpurun_out/it_ncu.log 2>&1; tail -2 gpurun_out/it_ncu.log
