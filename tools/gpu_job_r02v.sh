#!/bin/bash
# round 2: TMEM ring v2 (the 34 older ring loads in flight during the copy wait): correctness + A/B
mkdir -p gpurun_out/r02v
LB_PEER_TIMEOUT_MS=5000 LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_v2_ht122_pf2_e1_tmem1.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "two_step_kernel_bit" > gpurun_out/r02v/tests.log 2>&1; tail -1 gpurun_out/r02v/tests.log | cut -c1-300
TB_VARIANTS="default v2_ht104_pf3_e1_tmem1 v2_ht122_pf2_e1_tmem1" TB_REPS=1 TB_K=1000 bash tools/gpu_tb_ab.sh > gpurun_out/r02v/ab.log 2>&1; cat gpurun_out/r02v/ab.log
