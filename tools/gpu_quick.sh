#!/bin/bash
# quick GPU iteration: gpu tests + bench (+ optional extra command)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json | head -c 3000; tail -3 gpurun_out/bench.err
