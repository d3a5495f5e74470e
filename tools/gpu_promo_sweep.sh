#!/bin/bash
# Sweep of the two-step kernel's TMA L2 promotion: MLUPS (tb_bench) and ncu DRAM bytes per launch.
mkdir -p gpurun_out
TB_GRIDS=0 TB_L2=0 TB_PROMO=0,64,128,256 python tools/tb_bench.py > gpurun_out/promo.jsonl 2>&1
for p in 0 64 256; do
LB_TB_PROMO=$p ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_step2_tb -c 2 --csv --log-file gpurun_out/promo_ncu_$p.csv python tools/tb_ncu_target.py > /dev/null 2>&1
done
cat gpurun_out/promo.jsonl
grep -h "dram__bytes\|gpu__time" gpurun_out/promo_ncu_*.csv | awk -F'","' '{print $(NF-2), $NF}'
