#!/bin/bash
# One gpurun job: bench (both arms), launch list, ncu full captures of the hot kernels.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-extras > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_step2_tb|k_step_fused|k_propagate|k_collide|k_bc" \
    -s 0 -c 16 -o gpurun_out/prof_r01g -f python tools/ncu_target.py fused:bgk:tb fused split fused:regularized:tb fused:regularized split:regularized split:bgk:ldg > gpurun_out/ncu_full.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k 'regex:k_' --csv --log-file gpurun_out/ncu_metrics.csv python tools/ncu_target.py fused:bgk:tb fused:regularized:tb fused split fused:regularized split:regularized split:bgk:ldg fused:bgk:tma > gpurun_out/ncu_metrics.log 2>&1
ls -la gpurun_out
