#!/bin/bash
# One gpurun session: environment facts, microbenchmarks, GPU tests, benches.
set -x
mkdir -p gpurun_out
{ nvidia-smi; free -g; nproc; lscpu | head -20; python -c "import torch;print(torch.__version__, torch.cuda.get_device_name(0))"; } > gpurun_out/env.txt 2>&1
timeout 120 ./tools/microbench_atomics > gpurun_out/micro.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --maxfail=15 -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
tail -5 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --config rmat14 --steps 3 --warmup 3 --no-e2e --cpu-seconds 5 > gpurun_out/bench_rmat14.json 2> gpurun_out/bench_rmat14.err
timeout 1500 python bench.py --config rmat20 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_rmat20.json 2> gpurun_out/bench_rmat20.err
tail -3 gpurun_out/bench_rmat20.err
cat gpurun_out/bench_rmat20.json
