#!/bin/bash
# round 2: ISSUE2 (phase-2 warps refill the state-n buffers) and BGK-decoupled variants: correctness + A/B
mkdir -p gpurun_out/r02g
for v in issue23 issue23_decouple3; do
  LB_PEER_TIMEOUT_MS=5000 LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_ht104_pf1_e1_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "two_step" > gpurun_out/r02g/tests_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/r02g/tests_$v.log)"
done
LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_ht104_pf1_e1_decouple3_clock1.so timeout 300 python tools/tb_clock.py 1920 2048 gpurun_out/r02g/clock_decouple3.json > gpurun_out/r02g/clock_decouple3.log 2>&1; cut -c1-300 gpurun_out/r02g/clock_decouple3.log
TB_VARIANTS="default ht104_pf1_e1_issue23 ht104_pf1_e1_issue23_decouple3 ht104_pf1_e1_decouple3" TB_REPS=3 TB_K=1000 bash tools/gpu_tb_ab.sh > gpurun_out/r02g/ab.log 2>&1; cat gpurun_out/r02g/ab.log
