#!/bin/bash
# round 2: re-run the two failing GPU tests; per-CTA timelines (lead-in split vs none); A/B of variants
mkdir -p gpurun_out/r02f
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "injected_delay or n8_geometry or two_step" > gpurun_out/r02f/gpu_tests.log 2>&1; tail -3 gpurun_out/r02f/gpu_tests.log
for v in clock1 clock1_lead0; do
  LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_ht104_pf1_e1_$v.so timeout 300 python tools/tb_clock.py 1920 2048 gpurun_out/r02f/clock_$v.json > gpurun_out/r02f/clock_$v.log 2>&1
  echo "== $v"; cut -c1-400 gpurun_out/r02f/clock_$v.log
done
TB_VARIANTS="default ht104_pf1_e1_lead0 ht104_pf1_e1_nbar1 ht104_pf1_e1_decouple3" TB_REPS=2 TB_K=1000 bash tools/gpu_tb_ab.sh > gpurun_out/r02f/ab.log 2>&1; cat gpurun_out/r02f/ab.log
