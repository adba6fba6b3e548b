#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rmat20.csv python tools/run_once.py rmat20 > /dev/null 2>&1; python tools/ncu_summary.py gpurun_out/launches_rmat20.csv 5
SGB200_LIB=paper_2604_19004_b200/libsgb200_prof.so timeout 600 python tools/phase_prof.py rmat20 2>&1 | tail -10 | head -7
