#!/bin/bash
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rmat20.csv python tools/run_once.py rmat20 > gpurun_out/ncu_20.log 2>&1
python tools/ncu_summary.py gpurun_out/launches_rmat20.csv 14
