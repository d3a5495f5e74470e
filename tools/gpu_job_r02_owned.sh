#!/bin/bash
# round 2: phase 2 stores only owned rows (default) vs every computed row (variant), + the two-step / peer tests
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -x -q -k "two_step or peer or large or work_split" 2>&1 | tail -1
for rep in 1 2 3; do
  for v in default ht104_pf1_e1_store_owned0; do
    if [ "$v" = default ]; then unset LB_D2Q37_LIB; else export LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_$v.so; fi
    TB_K=1000 TB_GRIDS= TB_L2= TB_WT=0:0 timeout 300 python tools/tb_bench.py 2>&1 | grep tail_w16 | sed "s/^/$v /"
  done
done
