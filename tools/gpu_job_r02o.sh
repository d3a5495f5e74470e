#!/bin/bash
# round 2: HT = 108 with HT-row ring slots: parity (two-step tests) + A/B against the committed HT = 104 kernel
mkdir -p gpurun_out/r02o
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "two_step or peer_ring" > gpurun_out/r02o/tests.log 2>&1; tail -2 gpurun_out/r02o/tests.log
TB_VARIANTS="default head_ht104_pf1_e1 ht104_pf1_e1 ht100_pf1_e1" TB_REPS=2 TB_K=1000 bash tools/gpu_tb_ab.sh > gpurun_out/r02o/ab.log 2>&1; cat gpurun_out/r02o/ab.log
LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_ht108_pf1_e1_clock1.so timeout 300 python tools/tb_clock.py 1920 2048 gpurun_out/r02o/clock_ht108.json > gpurun_out/r02o/clock.log 2>&1; cut -c1-330 gpurun_out/r02o/clock.log
DET_CONFIGS=0:0 timeout 600 python tools/tb_determinism.py 1920 2048 1020 6 > gpurun_out/r02o/det.log 2>&1; cut -c1-300 gpurun_out/r02o/det.log
