#!/bin/bash
# round 2: clusters of 2 CTAs sweeping adjacent strips in lockstep (LB_TB_PAIR) and the aligned split (LB_TB_ALIGN)
# vs the default two-step kernel, A/B on one box, plus the two-step parity tests on the pair variant
mkdir -p gpurun_out
LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_ht104_pf1_e1_pair1.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_step or peer" > gpurun_out/pair_tests.log 2>&1
tail -3 gpurun_out/pair_tests.log
TB_REPS=3 TB_VARIANTS="default ht104_pf1_e1_pair1 ht104_pf1_e1_align1" bash tools/gpu_tb_ab.sh > gpurun_out/pair_ab.log 2>&1
cat gpurun_out/pair_ab.log
