#!/bin/bash
# round 2: full GPU suite + smoke + bench on the SKEW default; ncu full of the shipped kernel
O=gpurun_out/r02z
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; head -c 300 $O/bench.json; echo
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_step2_tb" -s 1 -c 1 -o $O/tb_full -f python tools/tb_ncu_target.py bgk > $O/ncu_full.log 2>&1; tail -1 $O/ncu_full.log
