#!/bin/bash
# A/B of two-step kernel variants on one box, long runs (sustained clocks / power), alternating.
for rep in $(seq ${TB_REPS:-2}); do
  for v in ${TB_VARIANTS:-default}; do
    if [ "$v" = default ]; then unset LB_D2Q37_LIB; else export LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_$v.so; fi
    echo "== $v rep $rep"
    TB_K=${TB_K:-2000} TB_GRIDS=0 TB_L2=0 timeout 300 python tools/tb_bench.py 2>&1 | sed -n '2p;4p'
  done
done
