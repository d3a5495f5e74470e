#!/bin/bash
# round 2: monitored pair path with PDL on the reduce kernel too: e2e breakdown with PDL on / off + monitor tests
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_long_run.py -m gpu -x -q -k "monitor or invariant or nonphys or nan or long" 2>&1 | tail -1
for rep in 1 2; do
  for pdl in 1 0; do
    TB_PDL=$pdl timeout 300 python tools/e2e_breakdown.py 1000 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$pdl', {k: d[k] for k in ['steps_plain_ms','steps_pair_monitored_ms','set_state_ms','gather_ms']})"
  done
done
