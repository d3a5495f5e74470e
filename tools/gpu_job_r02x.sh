#!/bin/bash
# round 2 final bench lines: default (config #2), configs #3 / #4 at N = 1, and the bench's N > 1 path on one GPU
O=gpurun_out/r02x
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; head -c 400 $O/bench.json; echo
timeout 900 python bench.py --config strong8192 --steps 100 --warmup 4 --no-extras > $O/bench_strong8192.json 2> $O/bench_strong8192.err; head -c 300 $O/bench_strong8192.json; echo
timeout 900 python bench.py --config weak4096 --steps 100 --warmup 4 --no-extras > $O/bench_weak4096.json 2> $O/bench_weak4096.err; head -c 300 $O/bench_weak4096.json; echo
LB_BENCH_SAME_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 4 --no-extras > $O/bench_same_gpu2.json 2> $O/bench_same_gpu2.err; head -c 600 $O/bench_same_gpu2.json; echo; tail -3 $O/bench_same_gpu2.err
