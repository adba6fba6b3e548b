#!/bin/bash
mkdir -p gpurun_out
for c in rmat17 rmat18; do
SGB200_LIB=paper_2604_19004_b200/libsgb200_prof.so timeout 600 python tools/phase_prof.py $c > gpurun_out/phase_$c.txt 2>&1
cat gpurun_out/phase_$c.txt
done
