mkdir -p gpurun_out
for v in "X=1" "SGB200_LIB=paper_2604_19004_b200/libsgb200_v8.so"; do
env $v timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; python -c "
import json; d=json.load(open('gpurun_out/it_bench.json')); print('$v', round(d['ms_per_step'],2), d['config']['stage_ms'], {k:v for k,v in d['roofline']['kernel_ms_per_step'].items()})"
for c in er10k poisson64; do
env $v timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; python -c "
import json; d=json.load(open('gpurun_out/it_bench.json')); print('$v $c', round(d['ms_per_step'],4), d['config']['stage_ms'])"
done
done
SGB200_LIB=paper_2604_19004_b200/libsgb200_v8.so timeout 600 python tools/timeline.py rmat20 2 > gpurun_out/timeline_rmat20.txt 2>&1; head -40 gpurun_out/timeline_rmat20.txt
SGB200_LIB=paper_2604_19004_b200/libsgb200_v8.so timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
SGB200_LIB=paper_2604_19004_b200/libsgb200_v8.so SANITIZE_ONLY=stress timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_cases.py > gpurun_out/rc_v8.txt 2>&1; grep -E "RACECHECK SUMMARY|sanitize cases ok" gpurun_out/rc_v8.txt; grep -A3 "Error: Potential" gpurun_out/rc_v8.txt | head -8
