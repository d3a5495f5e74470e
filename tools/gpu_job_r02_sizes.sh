#!/bin/bash
# round 2: aligned split (default, 0:0) vs contiguous split (19:1) at the bench size and configs #3 / #4
for rep in 1 2; do
  TB_K=1000 TB_GRIDS= TB_L2= TB_WT=0:0,19:1 timeout 300 python tools/tb_bench.py 1920 2048 2>&1 | grep tail_w16 | sed 's/^/1920x2048 /'
  TB_K=100 TB_GRIDS= TB_L2= TB_WT=0:0,19:1 timeout 600 python tools/tb_bench.py 4096 8192 2>&1 | grep tail_w16 | sed 's/^/4096x8192 /'
  TB_K=100 TB_GRIDS= TB_L2= TB_WT=0:0,19:1 timeout 900 python tools/tb_bench.py 8192 8192 2>&1 | grep tail_w16 | sed 's/^/8192x8192 /'
done
