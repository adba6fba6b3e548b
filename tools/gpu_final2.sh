mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/fin_pytest_gpu.txt; cat gpurun_out/fin_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; tail -c 600 gpurun_out/fin_bench.json
SAN_TIMEOUT=900 bash tools/sanitize.sh memcheck synccheck
SANITIZE_ONLY=stress timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_racecheck_stress.txt 2>&1; echo "racecheck(stress) rc=$? $(grep -E 'RACECHECK SUMMARY|sanitize cases ok' gpurun_out/sanitize_racecheck_stress.txt | tr '\n' ' ')"
