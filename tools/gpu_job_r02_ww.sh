#!/bin/bash
# round 2: wall-strip weight of the aligned split (BGK): per-CTA clocks and MLUPS per weight
mkdir -p gpurun_out/ww
for w in ${WWS:-19 22 24 26 28}; do
  TB_WW=$w LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_ht104_pf1_e1_clock1.so timeout 300 python tools/tb_clock.py 1920 2048 gpurun_out/ww/clock_ww$w.json > gpurun_out/ww/clock_ww$w.log 2>&1
done
for rep in 1 2; do
  TB_K=1000 TB_GRIDS= TB_L2= TB_WW=${WWB:-19,22,24,26,28,30} timeout 400 python tools/tb_bench.py 2>&1 | grep wall_w16
done
