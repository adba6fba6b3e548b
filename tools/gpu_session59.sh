#!/bin/bash
mkdir -p gpurun_out
L=$PWD/paper_2604_19004_b200
for lib in libsgb200_prof_nopf.so libsgb200_prof.so; do
echo "== $lib"; SGB200_LIB=$L/$lib timeout 600 python tools/phase_prof.py rmat20 2>&1 | tail -11
done
for lib in libsgb200_nopf.so libsgb200.so; do
SGB200_LIB=$L/$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_$lib.json 2> gpurun_out/b_$lib.err
python -c "import json,sys; d=json.loads(open('gpurun_out/b_$lib.json').read()); print('$lib', d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_step']['k_bmr'])"
done
