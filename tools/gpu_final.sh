#!/bin/bash
# Round-end evidence: GPU tests, default bench (with CPU baseline + e2e), reference arm,
# launch lists with DRAM traffic, full ncu captures of the dominant kernels.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json; tail -2 gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; cat gpurun_out/bench_reference.json
for c in poisson64 rect; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
bash tools/gpu_profiles.sh
