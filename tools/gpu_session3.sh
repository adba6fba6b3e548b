#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_warp -c 1 -o gpurun_out/prof_rect_hw python tools/run_once.py rect > gpurun_out/prof_rect.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_warp -c 1 -o gpurun_out/prof_poisson_hw python tools/run_once.py poisson64 > gpurun_out/prof_poisson.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bitmap -c 2 -o gpurun_out/prof_rmat16_bm python tools/run_once.py rmat16 > gpurun_out/prof_rmat16.log 2>&1
ls -la gpurun_out
