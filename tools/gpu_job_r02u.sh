#!/bin/bash
# round 2: ncu of the TMEM-ring variant
mkdir -p gpurun_out/r02u
LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_ht104_pf3_e1_tmem1.so timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_step2_tb" -s 1 -c 1 -o gpurun_out/r02u/tb_tmem -f python tools/tb_ncu_target.py bgk > gpurun_out/r02u/ncu.log 2>&1; tail -1 gpurun_out/r02u/ncu.log
TB_VARIANTS="ht104_pf2_e1_tmem1 ht122_pf2_e1_tmem1" TB_REPS=1 TB_K=1000 bash tools/gpu_tb_ab.sh > gpurun_out/r02u/ab.log 2>&1; cat gpurun_out/r02u/ab.log
