#!/bin/bash
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bitmap -c 1 -o gpurun_out/prof_bmc2 python tools/run_once.py rmat18 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hash_block -c 1 -o gpurun_out/prof_hb14 python tools/run_once.py rmat19 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep | tail -3
