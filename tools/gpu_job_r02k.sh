#!/bin/bash
# round 2: determinism stress of the two-step kernel (one bit_identical=false seen with L2 prefetch 4)
mkdir -p gpurun_out/r02k
timeout 900 python tools/tb_determinism.py 1920 2048 100 12 > gpurun_out/r02k/det.log 2>&1; cat gpurun_out/r02k/det.log | cut -c1-600
timeout 600 python tools/tb_determinism.py 1920 2048 1000 6 > gpurun_out/r02k/det1000.log 2>&1; cat gpurun_out/r02k/det1000.log | cut -c1-600
