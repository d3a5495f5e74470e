#!/bin/bash
# round 2: with SKEW the memory half binds: L2 prefetch distance sweep (LSU prefetch.global.L2) + skeleton variants
mkdir -p gpurun_out/r02aa
for rep in 1 2; do TB_K=1000 TB_GRIDS=0 TB_L2=0,1,2,3,4,6 timeout 600 python tools/tb_bench.py 2>&1 | grep '"tb": 1, "grid"'; done > gpurun_out/r02aa/l2.log; cat gpurun_out/r02aa/l2.log
TB_VARIANTS="default skew_ht104_pf1_e1_noload1 skew_ht104_pf1_e1_fake1" TB_REPS=1 TB_K=1000 bash tools/gpu_tb_ab.sh > gpurun_out/r02aa/ab.log 2>&1; cat gpurun_out/r02aa/ab.log
