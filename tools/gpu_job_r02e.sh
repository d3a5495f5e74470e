#!/bin/bash
# round 2: full gpu test suite (no -x) + ncu source-level capture of the two-step kernel
mkdir -p gpurun_out/r02e
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rs > gpurun_out/r02e/gpu_tests.log 2>&1; tail -15 gpurun_out/r02e/gpu_tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_step2_tb" -s 1 -c 1 -o gpurun_out/r02e/tb_src -f python tools/tb_ncu_target.py bgk > gpurun_out/r02e/ncu.log 2>&1
tail -2 gpurun_out/r02e/ncu.log
