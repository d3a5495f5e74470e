#!/bin/bash
# round 2: A/B of the strip height (HT = 108 default, 104 and 100 with HT-row ring slots) against the committed HT = 104 kernel
mkdir -p gpurun_out/r02p
TB_VARIANTS="default head_ht104_pf1_e1 ht104_pf1_e1 ht100_pf1_e1" TB_REPS=2 TB_K=1000 bash tools/gpu_tb_ab.sh > gpurun_out/r02p/ab.log 2>&1; cat gpurun_out/r02p/ab.log
