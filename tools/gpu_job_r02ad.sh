#!/bin/bash
# round 2: SKEW in one loop (phase 2's carried populations share phase 1's gather registers): tests, sanitizers, A/B
O=gpurun_out/r02ad
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x --timeout 600 -k "two_step or peer_ring or refill" > $O/tests.log 2>&1; tail -1 $O/tests.log
for tool in synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python tools/sanitize_target.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/sanitize_$tool.log | tail -1)"
done
TB_VARIANTS="default noskew_ht104_pf1_e1" TB_REPS=2 TB_K=1000 bash tools/gpu_tb_ab.sh > $O/ab.log 2>&1; cat $O/ab.log
