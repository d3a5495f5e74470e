#!/bin/bash
# round 2: ncu --set full of the FAKE skeleton (collision -> one multiply) of the two-step kernel; determinism stress (tb_bench protocol)
mkdir -p gpurun_out/r02l
LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_ht104_pf1_e1_fake1.so timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_step2_tb" -s 1 -c 1 -o gpurun_out/r02l/tb_fake -f python tools/tb_ncu_target.py bgk > gpurun_out/r02l/ncu.log 2>&1; tail -1 gpurun_out/r02l/ncu.log
DET_CONFIGS=0:0,0:4 timeout 900 python tools/tb_determinism.py 1920 2048 1020 16 > gpurun_out/r02l/det.log 2>&1; cut -c1-500 gpurun_out/r02l/det.log
