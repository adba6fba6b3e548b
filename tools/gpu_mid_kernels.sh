mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_hash_blockILi14ELi1E -c 1 -o gpurun_out/ev_full_hb14 -f python tools/run_once.py rmat20 > gpurun_out/ncu_hb14.log 2>&1; tail -2 gpurun_out/ncu_hb14.log
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_bitmapILi16384ELi1E -c 1 -o gpurun_out/ev_full_bm1 -f python tools/run_once.py rmat20 > gpurun_out/ncu_bm1.log 2>&1; tail -2 gpurun_out/ncu_bm1.log
ls -la gpurun_out/ev_full_hb14.ncu-rep gpurun_out/ev_full_bm1.ncu-rep
