#!/bin/bash
# round 2: ncu --set full of the NOLOAD (compute + stores) and NOLOAD+FAKE (skeleton without loads) variants
mkdir -p gpurun_out/r02s
for v in noload1 noload1_fake1; do
LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_ht104_pf1_e1_$v.so timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_step2_tb" -s 1 -c 1 -o gpurun_out/r02s/tb_$v -f python tools/tb_ncu_target.py bgk > gpurun_out/r02s/ncu_$v.log 2>&1; tail -1 gpurun_out/r02s/ncu_$v.log
done
