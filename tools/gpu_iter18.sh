mkdir -p gpurun_out
for v in "X=1" "SGB200_LIB=paper_2604_19004_b200/libsgb200_u12.so" "SGB200_LIB=paper_2604_19004_b200/libsgb200_u6.so"; do
env $v timeout 420 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; python -c "
import json; d=json.load(open('gpurun_out/it_bench.json')); print('$v', round(d['ms_per_step'],2), d['config']['stage_ms'], {k:v for k,v in d['roofline']['kernel_ms_per_step'].items()})"
done
