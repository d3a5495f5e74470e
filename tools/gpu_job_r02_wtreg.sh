#!/bin/bash
# round 2: the regularised two-step kernel with the aligned split: wall / tail weights (0:1 = contiguous default)
for rep in 1 2; do
  TB_WT_COLL=regularized TB_K=1000 TB_GRIDS= TB_L2= TB_WT=${WT:-0:1,20:16,20:17,21:17,22:17,22:18,24:17} timeout 600 python tools/tb_bench.py 2>&1 | grep tail_w16
done
