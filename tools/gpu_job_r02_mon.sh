#!/bin/bash
# round 2: monitored two-step kernel, branch-free hook (default) vs branched (variant), e2e breakdown A/B + monitor tests
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -x -q -k "monitor or invariant or nonphys or nan" 2>&1 | tail -1
for rep in 1 2; do
  for v in default ht104_pf1_e1_mon_branchless0; do
    if [ "$v" = default ]; then unset LB_D2Q37_LIB; else export LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_$v.so; fi
    timeout 300 python tools/e2e_breakdown.py 1000 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', {k: d[k] for k in ['steps_plain_ms','steps_pair_monitored_ms','profile_pair_monitored_200']})"
  done
done
