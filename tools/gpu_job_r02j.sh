#!/bin/bash
# round 2: TMA L2 prefetch of whole column windows (LB_OPT_TB_L2_PREFETCH distance sweep), correctness first
mkdir -p gpurun_out/r02j
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "two_step" > gpurun_out/r02j/tests.log 2>&1; tail -1 gpurun_out/r02j/tests.log
for rep in 1 2; do TB_K=1000 TB_GRIDS=0 TB_L2=0,2,3,4,6,8,12,16 timeout 600 python tools/tb_bench.py 2>&1 | grep '"tb": 1, "grid"'; done > gpurun_out/r02j/l2.log; cat gpurun_out/r02j/l2.log
