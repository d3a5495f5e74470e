#!/bin/bash
# round 2: in-kernel N > 1 exchange reading the neighbours' buffers by TMA + in-kernel signal: tests, ring timeline, timing model, config #5 N = 8
mkdir -p gpurun_out/r02r
O=gpurun_out/r02r
LB_PEER_TIMEOUT_MS=5000 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ipc.py tests/test_gpu_long_run.py tests/test_gpu_large.py -q -x --timeout 600 -k "peer or ring or ipc or two_step or n8 or nccl" > $O/tests.log 2>&1; tail -3 $O/tests.log
timeout 900 python tools/ring_timeline.py --n 4 --lx 1920 --ly 2048 --pairs 50 --out $O/r02_ring_timeline.json > $O/ring.log 2>&1; tail -4 $O/ring.log | cut -c1-700
timeout 900 python tools/timing_model_tb.py --out $O/r02_timing_model.json > $O/tm.log 2>&1; tail -3 $O/tm.log | cut -c1-900
timeout 1500 python tests/long_run.py --lx 2048 --ly 4096 --nslabs 8 --compare-n1 --steps 10000 --every 100 --ckpt-every 1000 --check 10 --out $O/r02_long_run_n8.json > $O/lr.log 2>&1; tail -1 $O/lr.log | cut -c1-700
