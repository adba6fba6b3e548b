#!/bin/bash
# Evidence capture for profiles/: launch lists (time + DRAM) and one full
# ncu capture of the dominant kernel.  1 GPU.
mkdir -p gpurun_out
for c in rmat20 poisson64 rect; do
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python tools/run_once.py $c > /dev/null 2>&1
done
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_bmr -c 2 -o gpurun_out/full_k_bmr_rmat20 python tools/run_once.py rmat20 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_escr -c 1 -o gpurun_out/full_escr_rect python tools/run_once.py rect > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep | tail -3
