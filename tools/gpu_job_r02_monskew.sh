#!/bin/bash
# round 2: monitored pair path — default (SKEW) vs the SKEW-free variant
for rep in 1 2; do
  for v in default ht104_pf1_e1_skew0; do
    if [ "$v" = default ]; then unset LB_D2Q37_LIB; else export LB_D2Q37_LIB=$PWD/paper_1703_00186_b200/variants/liblb_$v.so; fi
    timeout 300 python tools/e2e_breakdown.py 1000 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', {k: d[k] for k in ['steps_plain_ms','steps_pair_monitored_ms']})"
  done
done
