#!/bin/bash
# round 2: late ISSUE2 variant A/B; wall-weight sweep of the default build (BGK)
mkdir -p gpurun_out/r02h
TB_VARIANTS="default ht104_pf1_e1_issue21_issue2_late1" TB_REPS=2 TB_K=1000 bash tools/gpu_tb_ab.sh > gpurun_out/r02h/ab.log 2>&1; cat gpurun_out/r02h/ab.log
for rep in 1 2; do TB_K=1000 TB_GRIDS= TB_L2= TB_WW=18,19,20,17,21 timeout 300 python tools/tb_bench.py 2>&1 | grep wall_w16; done > gpurun_out/r02h/ww.log; cat gpurun_out/r02h/ww.log
