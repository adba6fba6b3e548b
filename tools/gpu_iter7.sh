mkdir -p gpurun_out
for v in "X=1" "SGB200_LIB=paper_2604_19004_b200/libsgb200_v1.so" "SGB200_LIB=paper_2604_19004_b200/libsgb200_v2.so"; do
env $v timeout 900 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; python -c "
import json; d=json.load(open('gpurun_out/it_bench.json')); print('$v', round(d['ms_per_step'],2), d['config']['stage_ms'])"
done
SG_BENCH_SAME_DEVICE=1 SG_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config rmat16 --steps 2 --warmup 1 --batch-products 1e8 --no-e2e > gpurun_out/n2_batched.json 2> gpurun_out/n2_batched.err; tail -c 1500 gpurun_out/n2_batched.json; tail -3 gpurun_out/n2_batched.err
