#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --maxfail=10 -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
tail -5 gpurun_out/pytest_gpu.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bmw -c 1 -o gpurun_out/prof_bmw_rmat18 python tools/run_once.py rmat18 > gpurun_out/prof_bmw.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bitmap -c 1 -o gpurun_out/prof_bmc_rmat18 python tools/run_once.py rmat18 > gpurun_out/prof_bmc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_warp -c 1 -o gpurun_out/prof_rect_hw python tools/run_once.py rect > gpurun_out/prof_rect.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hash_block -c 1 -o gpurun_out/prof_hb_rmat18 python tools/run_once.py rmat18 > gpurun_out/prof_hb.log 2>&1
ls -la gpurun_out/*.ncu-rep
