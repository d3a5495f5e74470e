#!/bin/bash
# round 2: programmatic dependent launch of the two-step kernel on / off, alternating, plus the two-step tests
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_step or peer" 2>&1 | tail -1
for rep in 1 2 3; do
  for pdl in 1 0; do
    TB_PDL=$pdl TB_K=1000 TB_GRIDS= TB_L2= TB_WT=0:0 timeout 300 python tools/tb_bench.py 2>&1 | grep tail_w16 | sed "s/^/pdl=$pdl K=1000 /"
    TB_PDL=$pdl TB_K=20 TB_GRIDS= TB_L2= TB_WT=0:0 timeout 300 python tools/tb_bench.py 2>&1 | grep tail_w16 | sed "s/^/pdl=$pdl K=20 /"
  done
done
