#!/bin/bash
# round 2: wall / tail weights at configs #3 / #4 sizes (BGK, K = 100)
for rep in 1 2; do
  TB_K=100 TB_GRIDS= TB_L2= TB_WT=0:0,21:16,21:18,21:20,19:17,23:17 timeout 900 python tools/tb_bench.py 8192 8192 2>&1 | grep tail_w16 | sed 's/^/8192x8192 /'
  TB_K=100 TB_GRIDS= TB_L2= TB_WT=0:0,21:16,21:18,21:20,19:17,23:17 timeout 900 python tools/tb_bench.py 4096 8192 2>&1 | grep tail_w16 | sed 's/^/4096x8192 /'
done
