#!/bin/bash
# round 2 final: full GPU suite, smoke, then the evidence job (bench both arms, launch list, ncu metrics + full, sanitizers)
O=${O:-gpurun_out/r02final}
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
O=$O bash tools/gpu_bench_round_r02.sh
