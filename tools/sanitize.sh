#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over tools/sanitize_cases.py and
# smoke(); logs in gpurun_out/sanitize_<tool>.log.
mkdir -p gpurun_out
CS=$(command -v compute-sanitizer || echo /usr/local/cuda/bin/compute-sanitizer)
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --error-exitcode 17 python tools/sanitize_cases.py \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
done
timeout 900 $CS --tool memcheck --error-exitcode 17 python __graft_entry__.py smoke > gpurun_out/sanitize_smoke.log 2>&1
echo "smoke memcheck rc=$?" >> gpurun_out/sanitize_summary.txt
