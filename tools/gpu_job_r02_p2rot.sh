#!/bin/bash
# round 2: phase-2 warp rotation (LB_TB_P2ROT: default 2 vs variants 0 / 1) x wall weight, A/B on one box
for rep in 1 2; do
  for v in default ht104_pf1_e1_p2rot0 ht104_pf1_e1_p2rot1; do
    if [ "$v" = default ]; then unset LB_D2Q37_LIB; else export LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_$v.so; fi
    TB_K=1000 TB_GRIDS= TB_L2= TB_WT=0:0,19:17,20:17 timeout 300 python tools/tb_bench.py 2>&1 | grep tail_w16 | sed "s/^/$v /"
    TB_WT_COLL=regularized TB_K=1000 TB_GRIDS= TB_L2= TB_WT=0:0 timeout 300 python tools/tb_bench.py 2>&1 | grep tail_w16 | sed "s/^/$v /"
  done
done
