mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_scale.py -m gpu -q -x 2>&1 | tail -1
timeout 420 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; python -c "
import json; d=json.load(open('gpurun_out/it_bench.json')); print(round(d['ms_per_step'],2), d['config']['stage_ms'])"
for c in er10k poisson64 rect; do
timeout 420 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; python -c "
import json; d=json.load(open('gpurun_out/it_bench.json')); print('$c', round(d['ms_per_step'],4), d['config']['stage_ms'])"
done
