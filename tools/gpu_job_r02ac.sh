#!/bin/bash
# round 2: does prefetch depth lift the memory half?  FAKE skeleton at HT 88 with 2 vs 3 state-n buffers
O=gpurun_out/r02ac
mkdir -p $O
TB_VARIANTS="dp_ht88_pf1_e1_fake1 dp_ht88_pf2_e1_fake1" TB_REPS=2 TB_K=1000 bash tools/gpu_tb_ab.sh > $O/ab.log 2>&1; cat $O/ab.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "two_step or peer_ring" > $O/tests.log 2>&1; tail -1 $O/tests.log
for tool in synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python tools/sanitize_target.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/sanitize_$tool.log | tail -1)"
done
TB_VARIANTS="default" TB_REPS=2 TB_K=1000 bash tools/gpu_tb_ab.sh > $O/ab_default.log 2>&1; cat $O/ab_default.log
