#!/bin/bash
# Two-step kernel tiling variants (tools/build_tb_variant.py): MLUPS + bit identity (tb_bench),
# and the two-step parity tests, per variant library.
mkdir -p gpurun_out
for v in ${TB_VARIANTS:-default}; do
  if [ "$v" = default ]; then unset LB_D2Q37_LIB; else export LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_$v.so; fi
  echo "== $v"
  TB_GRIDS=0 TB_L2=0 timeout 300 python tools/tb_bench.py 2>&1 | tail -4
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "two_step" 2>&1 | tail -2
done
