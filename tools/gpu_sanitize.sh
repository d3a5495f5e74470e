#!/bin/bash
# compute-sanitizer passes over tools/sanitize_target.py (summaries to gpurun_out/)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python tools/sanitize_target.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
