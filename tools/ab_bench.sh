#!/bin/bash
# A/B of library builds (RK_LIB) on bench lines: bash tools/ab_bench.sh "<lib1> <lib2> ..." "<workloads>" "<dtypes>" [reps]
LIBS=$1; WLS=${2:-par512}; DTS=${3:-fp32}; REPS=${4:-1}
for r in $(seq 1 $REPS); do for L in $LIBS; do for wl in $WLS; do for dt in $DTS; do
  RK_LIB=$L timeout 300 python bench.py --workload $wl --dtype $dt --no-cpu-baseline --no-extras --no-e2e --no-parity 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); pk=d['roofline']['per_kernel']
print('$L $wl $dt', round(d['value']), 'fwd', round(pk['forward']['ms'],3), 'bp', round(pk['backproject']['ms'],3))"
done; done; done; done
