#!/bin/bash
# compute-sanitizer over the small parity cases (tools/sanitize_cases.py):
# memcheck (out-of-bounds / misaligned / leaks), racecheck (shared-memory
# hazards), synccheck (illegal barrier use), initcheck (uninitialised global
# reads).  Logs go to gpurun_out/sanitize_<tool>.txt (summaries in profiles/).
mkdir -p gpurun_out
# tools to run: arguments (default all four)
TOOLS="${@:-memcheck racecheck synccheck initcheck}"
for tool in $TOOLS; do
  extra=""
  # (no leak check: the torch caching allocator keeps its pool until exit by design)
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout ${SAN_TIMEOUT:-3000} compute-sanitizer --tool $tool $extra --print-limit 200 --error-exitcode 9 \
      python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases ok' gpurun_out/sanitize_$tool.txt | tr '\n' ' ')"
done
