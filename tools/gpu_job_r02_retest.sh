#!/bin/bash
# round 2: earlier-rejected two-step variants re-tested on the aligned-split kernel (BGK + regularised), alternating
for rep in 1 2; do
  for v in default ht104_pf1_e1_decouple3 ht104_pf1_e1_nbar1 ht104_pf1_e1_lead5 ht104_pf1_e1_lead9 ht104_pf1_e1_skew3_decouple0; do
    if [ "$v" = default ]; then unset LB_D2Q37_LIB; else export LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_$v.so; fi
    TB_K=1000 TB_GRIDS= TB_L2= TB_WT=0:0 timeout 300 python tools/tb_bench.py 2>&1 | grep tail_w16 | sed "s/^/$v /"
    TB_WT_COLL=regularized TB_K=1000 TB_GRIDS= TB_L2= TB_WT=0:0 timeout 300 python tools/tb_bench.py 2>&1 | grep tail_w16 | sed "s/^/$v /"
  done
done
for promo in 0 256; do TB_PROMO=$promo TB_K=1000 TB_GRIDS= TB_L2= timeout 300 python tools/tb_bench.py 2>&1 | grep l2_promotion; done
