#!/bin/bash
# round 2: hunt the first differing two-step launch (seen with TMA L2 prefetch 4), then the default
mkdir -p gpurun_out/r02m
timeout 900 python tools/tb_race_hunt.py 1920 2048 500 8 4 > gpurun_out/r02m/hunt4.log 2>&1; cut -c1-1500 gpurun_out/r02m/hunt4.log
timeout 600 python tools/tb_race_hunt.py 1920 2048 500 6 0 > gpurun_out/r02m/hunt0.log 2>&1; cut -c1-1500 gpurun_out/r02m/hunt0.log
