#!/bin/bash
# round 2 re-entry: verify the committed tree on a B200 (gpu tests, bench, launch list)
mkdir -p gpurun_out/r02d
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02d/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -rs > gpurun_out/r02d/gpu_tests.log 2>&1; tail -5 gpurun_out/r02d/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d/smoke.log 2>&1; tail -2 gpurun_out/r02d/smoke.log
timeout 300 python bench.py > gpurun_out/r02d/bench.json 2> gpurun_out/r02d/bench.err; head -c 2500 gpurun_out/r02d/bench.json; tail -3 gpurun_out/r02d/bench.err
