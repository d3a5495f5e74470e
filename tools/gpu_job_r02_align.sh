#!/bin/bash
# round 2: time-aligned work split of the two-step kernel (LB_TB_ALIGN variant) vs the default, A/B on one box
mkdir -p gpurun_out
TB_REPS=3 TB_VARIANTS="default ht104_pf1_e1_align1" bash tools/gpu_tb_ab.sh > gpurun_out/align_ab.log 2>&1
LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_ht104_pf1_e1_align1.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_step" > gpurun_out/align_tests.log 2>&1
tail -3 gpurun_out/align_tests.log
cat gpurun_out/align_ab.log
