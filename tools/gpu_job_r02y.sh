#!/bin/bash
# round 2: SKEW (phase 2 offset within the iteration): correctness + A/B
mkdir -p gpurun_out/r02y
for v in ht104_pf1_e1_skew1 ht104_pf1_e1_skew3_decouple0; do
LB_PEER_TIMEOUT_MS=5000 LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "two_step or peer_ring" > gpurun_out/r02y/tests_$v.log 2>&1; echo "$v $(tail -1 gpurun_out/r02y/tests_$v.log | cut -c1-200)"
done
TB_VARIANTS="default ht104_pf1_e1_skew1 ht104_pf1_e1_skew3_decouple0" TB_REPS=2 TB_K=1000 bash tools/gpu_tb_ab.sh > gpurun_out/r02y/ab.log 2>&1; cat gpurun_out/r02y/ab.log
