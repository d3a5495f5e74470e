#!/bin/bash
# round 2 final evidence on the aligned-split + PDL kernel: GPU tests, smoke, bench lines (K = 1000 default, the
# driver's K = 20, configs #3 / #4), reference arm, ncu launch list, ncu metrics, --set full of k_step2_tb
O=${O:-gpurun_out/r02final4}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; head -c 200 $O/bench.json; echo
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_k20.json 2> $O/bench_k20.err
for c in strong8192 weak4096; do timeout 900 python bench.py --config $c --steps 100 --warmup 4 > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-extras > $O/launches_bench.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k 'regex:k_' --csv --log-file $O/ncu_metrics.csv python tools/ncu_target.py fused:bgk:tb fused:regularized:tb fused split fused:regularized split:regularized split:bgk:ldg fused:bgk:tma > $O/ncu_metrics.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_step2_tb" -s 1 -c 1 -o $O/tb_full -f python tools/tb_ncu_target.py bgk > $O/ncu_full.log 2>&1
ls $O
