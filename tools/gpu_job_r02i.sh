#!/bin/bash
# round 2: the two-step kernel's data-movement skeleton (LB_TB_FAKE: collision -> one multiply) timing + per-CTA clocks; wall-weight sweep
mkdir -p gpurun_out/r02i
TB_VARIANTS="default ht104_pf1_e1_fake1" TB_REPS=2 TB_K=1000 bash tools/gpu_tb_ab.sh > gpurun_out/r02i/ab.log 2>&1; cat gpurun_out/r02i/ab.log
LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_ht104_pf1_e1_fake1_clock1.so timeout 300 python tools/tb_clock.py 1920 2048 gpurun_out/r02i/clock_fake.json > gpurun_out/r02i/clock_fake.log 2>&1; cut -c1-300 gpurun_out/r02i/clock_fake.log
for rep in 1 2; do TB_K=1000 TB_GRIDS= TB_L2= TB_WW=18,19,20,17,21 timeout 300 python tools/tb_bench.py 2>&1 | grep wall_w16; done > gpurun_out/r02i/ww.log; cat gpurun_out/r02i/ww.log
