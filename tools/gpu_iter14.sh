mkdir -p gpurun_out
SGB200_LIB=paper_2604_19004_b200/libsgb200_nobulk.so SAN_TIMEOUT=1800 bash tools/sanitize.sh initcheck
SGB200_LIB=paper_2604_19004_b200/libsgb200_nobulk.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
timeout 420 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; python -c "
import json; d=json.load(open('gpurun_out/it_bench.json')); print(round(d['ms_per_step'],2), d['config']['stage_ms'])"
