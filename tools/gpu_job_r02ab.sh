#!/bin/bash
# round 2: the cross-proxy write-after-read (phase-1 gather LDS vs TMA refill of the same buffer): stress with L2 prefetch
# (fast refills), with and without the proxy fence; then the short ring at HT 114 / 104 (SKEW) A/B
O=gpurun_out/r02ab
mkdir -p $O
for rep in 1 2 3; do TB_K=1000 TB_GRIDS=0 TB_L2=0,1,2,3,4 timeout 600 python tools/tb_bench.py 2>&1 | grep '"tb": 1, "grid"'; done > $O/fence_l2.log; echo "fence:"; cat $O/fence_l2.log | cut -c1-160
for rep in 1 2; do LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_ht104_pf1_e1_war_fence0.so TB_K=1000 TB_GRIDS=0 TB_L2=0,1,2,3 timeout 600 python tools/tb_bench.py 2>&1 | grep '"tb": 1, "grid"'; done > $O/nofence_l2.log; echo "no fence:"; cat $O/nofence_l2.log | cut -c1-160
for v in ht114_pf1_e1_shortring1_skew3_decouple0 ht104_pf1_e1_shortring1_skew3_decouple0; do
LB_PEER_TIMEOUT_MS=5000 LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "two_step_kernel_bit and bgk" > $O/tests_$v.log 2>&1; echo "$v $(tail -1 $O/tests_$v.log | cut -c1-200)"
done
TB_VARIANTS="default ht104_pf1_e1_war_fence0 ht114_pf1_e1_shortring1_skew3_decouple0 ht104_pf1_e1_shortring1_skew3_decouple0" TB_REPS=2 TB_K=1000 bash tools/gpu_tb_ab.sh > $O/ab.log 2>&1; cat $O/ab.log
