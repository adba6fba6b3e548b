#!/bin/bash
# Round evidence on one B200: GPU tests, benches (default R-MAT-20 with e2e,
# CPU reference and parity; the other configs; FORCE_ESTIMATE), the reference
# arm, ncu launch lists with DRAM traffic and one full ncu capture of k_win.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,driver_version --format=csv > gpurun_out/ev_smi.txt; nproc >> gpurun_out/ev_smi.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.txt 2>&1; tail -2 gpurun_out/ev_pytest_gpu.txt
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/ev_bench_rmat20.json 2> gpurun_out/ev_bench_rmat20.err; tail -c 400 gpurun_out/ev_bench_rmat20.json; echo
timeout 1200 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/ev_bench_reference.json 2> gpurun_out/ev_bench_reference.err; tail -c 300 gpurun_out/ev_bench_reference.json; echo
for c in poisson64 er10k; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --parity-blocks 1 > gpurun_out/ev_bench_$c.json 2> gpurun_out/ev_bench_$c.err; tail -c 200 gpurun_out/ev_bench_$c.json; echo
done
timeout 900 python bench.py --config rect --steps 10 --warmup 3 --no-cpu > gpurun_out/ev_bench_rect.json 2> gpurun_out/ev_bench_rect.err; tail -c 200 gpurun_out/ev_bench_rect.json; echo
timeout 900 python bench.py --workflow estimate --steps 5 --warmup 2 --no-e2e --no-cpu > gpurun_out/ev_bench_estimate.json 2> gpurun_out/ev_bench_estimate.err; tail -c 200 gpurun_out/ev_bench_estimate.json; echo
for c in rmat20 poisson64 rect; do
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev_launches_$c.csv python tools/run_once.py $c > /dev/null 2>&1
done
timeout 1200 ncu --set full --clock-control none --import-source on -k k_win -c 1 -o gpurun_out/ev_full_k_win -f python tools/run_once.py rmat20 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_bitmap -c 1 -o gpurun_out/ev_full_count -f python tools/run_once.py rmat20 > /dev/null 2>&1
ls -la gpurun_out/ev_*
SAN_TIMEOUT=900 bash tools/sanitize.sh memcheck synccheck
SANITIZE_ONLY=stress timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_racecheck_stress.txt 2>&1; echo "racecheck(stress) rc=$? $(grep -E 'RACECHECK SUMMARY|sanitize cases ok' gpurun_out/sanitize_racecheck_stress.txt | tr '\n' ' ')"
