#!/bin/bash
# round 2 measurements on the shipped kernels: N > 1 exchange timeline, timing model refit,
# config #5 at its N = 8 geometry (10^4 steps), drift study, FP64 peak with NVML clocks
mkdir -p gpurun_out/r02q
O=gpurun_out/r02q
timeout 900 python tools/ring_timeline.py --n 4 --lx 1920 --ly 2048 --pairs 50 --out $O/r02_ring_timeline.json > $O/ring.log 2>&1; tail -4 $O/ring.log | cut -c1-600
timeout 900 python tools/timing_model_tb.py --out $O/r02_timing_model.json > $O/tm.log 2>&1; tail -3 $O/tm.log | cut -c1-800
timeout 1500 python tests/long_run.py --lx 2048 --ly 4096 --nslabs 8 --compare-n1 --steps 10000 --every 100 --ckpt-every 1000 --check 10 --out $O/r02_long_run_n8.json > $O/lr.log 2>&1; tail -2 $O/lr.log | cut -c1-1200
timeout 1200 python tools/drift_study.py --lx 256 --ly 4096 --steps 1000 --every 100 --side both --out $O/r02_drift_study.json > $O/drift.log 2>&1; tail -4 $O/drift.log | cut -c1-800
timeout 300 python tools/fp64_bench.py --out $O/r02_fp64_hbm_microbench.json > $O/fp64.log 2>&1; tail -3 $O/fp64.log | cut -c1-600
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
