#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
for c in rmat18; do
SGB200_LIB=paper_2604_19004_b200/libsgb200_prof.so timeout 600 python tools/phase_prof.py $c > gpurun_out/phase_$c.txt 2>&1
tail -12 gpurun_out/phase_$c.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rmat18.csv python tools/run_once.py rmat18 > gpurun_out/ncu_b.log 2>&1
python tools/ncu_summary.py gpurun_out/launches_rmat18.csv 6
