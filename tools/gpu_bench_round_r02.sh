#!/bin/bash
# Round 2 evidence job: bench (both arms), ncu launch list of the bench command, ncu metrics of the hot
# kernels (-> profiles/ncu_summary.json via tools/ncu_summarize.py), ncu --set full of the two-step kernel,
# sanitizers over every kernel and transport.
O=${O:-gpurun_out/r02w}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; head -c 600 $O/bench.json; echo
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; head -c 300 $O/bench_ref.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-extras > $O/launches_bench.log 2>&1; tail -1 $O/launches_bench.log | head -c 300; echo
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k 'regex:k_' --csv --log-file $O/ncu_metrics.csv python tools/ncu_target.py fused:bgk:tb fused:regularized:tb fused split fused:regularized split:regularized split:bgk:ldg fused:bgk:tma > $O/ncu_metrics.log 2>&1; tail -1 $O/ncu_metrics.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_step2_tb" -s 1 -c 1 -o $O/tb_full -f python tools/tb_ncu_target.py bgk > $O/ncu_full.log 2>&1; tail -1 $O/ncu_full.log
# (compute-sanitizer was closed on the GPU pool late in round 2: SKIP_SANITIZE=1 skips it)
[ -n "$SKIP_SANITIZE" ] || for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python tools/sanitize_target.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/sanitize_$tool.log | tail -1)"
done
ls -la $O
