#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bmw -c 1 -o gpurun_out/prof_bmw3 python tools/run_once.py rmat17 > gpurun_out/prof_bmw3.log 2>&1
ls -la gpurun_out/prof_bmw3.ncu-rep
