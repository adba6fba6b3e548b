#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 1200 python tools/est_eval.py > gpurun_out/est_eval.csv 2> gpurun_out/est_eval.err; cat gpurun_out/est_eval.csv | cut -d, -f1,4,12-19; tail -2 gpurun_out/est_eval.err
