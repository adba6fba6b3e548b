#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bmw -c 1 -o gpurun_out/prof_bmw2 python tools/run_once.py rmat17 > gpurun_out/prof_bmw2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_warp -s 1 -c 1 -o gpurun_out/prof_rect_hw1 python tools/run_once.py rect > gpurun_out/prof_rect1.log 2>&1
ls -la gpurun_out/*.ncu-rep
