#!/bin/bash
# round 2: TMEM-resident state-(n+1) ring (LB_TB_TMEM, 4 state-n buffers): correctness then A/B
mkdir -p gpurun_out/r02t
V=$PWD/paper_1703_00186_b200/variants/liblb_ht104_pf3_e1_tmem1.so
LB_PEER_TIMEOUT_MS=5000 LB_D2Q37_LIB=$V timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "two_step_kernel_bit" > gpurun_out/r02t/tests.log 2>&1; tail -15 gpurun_out/r02t/tests.log | cut -c1-300
LB_D2Q37_LIB=$V DET_CONFIGS=0:0 timeout 300 python tools/tb_determinism.py 1920 2048 100 2 > gpurun_out/r02t/det.log 2>&1; cut -c1-400 gpurun_out/r02t/det.log
TB_VARIANTS="default ht104_pf3_e1_tmem1" TB_REPS=2 TB_K=1000 bash tools/gpu_tb_ab.sh > gpurun_out/r02t/ab.log 2>&1; cat gpurun_out/r02t/ab.log
