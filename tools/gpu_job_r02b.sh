#!/bin/bash
# round 2: full gpu tests on the default build, named-barrier variants: two-step tests + A/B
mkdir -p gpurun_out/r02b
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02b/gpu_tests.log 2>&1; tail -3 gpurun_out/r02b/gpu_tests.log
for v in ht104_pf1_e1_nbar1 ht104_pf1_e1_nbar3_decouple0; do
  LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "two_step" > gpurun_out/r02b/tests_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/r02b/tests_$v.log)"
done
TB_VARIANTS="default ht104_pf1_e1_nbar1 ht104_pf1_e1_nbar3_decouple0" TB_REPS=2 bash tools/gpu_tb_ab.sh > gpurun_out/r02b/ab.log 2>&1; cat gpurun_out/r02b/ab.log
