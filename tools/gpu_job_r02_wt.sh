#!/bin/bash
# round 2: wall and tail weights of the aligned split (BGK): MLUPS per (wall, tail) and per-CTA clocks
mkdir -p gpurun_out/wt
for rep in 1 2; do
  TB_K=1000 TB_GRIDS= TB_L2= TB_WT=${WT:-19:16,21:16,21:17,21:18,21:19,22:17,22:18,26:16} timeout 600 python tools/tb_bench.py 2>&1 | grep tail_w16
done
for c in ${WTC:-21:18 22:18}; do
  w=${c%:*}; t=${c#*:}
  TB_WW=$w TB_TW=$t LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_ht104_pf1_e1_clock1.so timeout 300 python tools/tb_clock.py 1920 2048 gpurun_out/wt/clock_${w}_${t}.json > gpurun_out/wt/clock_${w}_${t}.log 2>&1
done
