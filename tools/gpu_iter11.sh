mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; python -c "
import json; d=json.load(open('gpurun_out/it_bench.json')); print(round(d['ms_per_step'],2), d['config']['stage_ms'], {k:v for k,v in d['roofline']['kernel_ms_per_step'].items()})"
SANITIZE_ONLY=stress timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_cases.py > gpurun_out/rc_main.txt 2>&1; grep -E "RACECHECK SUMMARY|sanitize cases ok" gpurun_out/rc_main.txt; grep -A3 "Error: Potential" gpurun_out/rc_main.txt | head -8
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
