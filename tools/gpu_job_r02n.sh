#!/bin/bash
# round 2: race hunt (first differing two-step launch); compute-only (NOLOAD) variants timing
mkdir -p gpurun_out/r02n
timeout 900 python tools/tb_race_hunt.py 1920 2048 500 8 4 > gpurun_out/r02n/hunt4.log 2>&1; cut -c1-1500 gpurun_out/r02n/hunt4.log
TB_VARIANTS="default ht104_pf1_e1_noload1 ht104_pf1_e1_noload1_fake1 ht104_pf1_e1_fake1" TB_REPS=1 TB_K=1000 bash tools/gpu_tb_ab.sh > gpurun_out/r02n/ab.log 2>&1; cat gpurun_out/r02n/ab.log
timeout 600 python tools/tb_race_hunt.py 1920 2048 500 8 0 > gpurun_out/r02n/hunt0.log 2>&1; cut -c1-1500 gpurun_out/r02n/hunt0.log
