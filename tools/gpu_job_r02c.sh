#!/bin/bash
# round 2: gpu tests on the default build; two-step variants (named-barrier hand-over, FP64-free skeleton): correctness + A/B
mkdir -p gpurun_out/r02c
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/r02c/gpu_tests.log 2>&1; tail -3 gpurun_out/r02c/gpu_tests.log
for v in ht104_pf1_e1_nbar1 ht104_pf1_e1_nbar3_decouple0; do
  LB_PEER_TIMEOUT_MS=5000 LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "two_step_kernel_bit or two_step_kernel_grid or two_step_kernel_monitors" > gpurun_out/r02c/tests_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/r02c/tests_$v.log)"
done
for rep in 1 2; do
  for v in default ht104_pf1_e1_nbar1 ht104_pf1_e1_nbar3_decouple0 ht104_pf1_e1_fake1; do
    if [ "$v" = default ]; then unset LB_D2Q37_LIB; else export LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_$v.so; fi
    echo "== $v rep $rep"
    TB_K=1000 TB_GRIDS=0 TB_L2=0 timeout 120 python tools/tb_bench.py 2>&1 | sed -n '2p;4p'
  done
done > gpurun_out/r02c/ab.log 2>&1; cat gpurun_out/r02c/ab.log
