#!/bin/bash
# A/B of an env setting on bench lines: bash ab_env.sh "<VAR=a> <VAR=b>" "<workloads>" "<dtypes>" reps
for r in $(seq 1 ${4:-1}); do for E in $1; do for wl in $2; do for dt in $3; do
  env $E timeout 300 python bench.py --workload $wl --dtype $dt --no-cpu-baseline --no-extras --no-e2e --no-parity 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); pk=d['roofline']['per_kernel']
print('$E $wl $dt', round(d['value']), 'fwd', round(pk['forward']['ms'],3), 'bp', round(pk['backproject']['ms'],3))"
done; done; done; done
