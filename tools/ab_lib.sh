#!/bin/bash
# A/B of two library builds (RK_LIB): bench lines + ncu counters of the forward kernel.
# Usage (under gpurun): bash tools/ab_lib.sh <libA> <libB> [workload]
WL=${3:-par512}
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
for L in "$1" "$2"; do
  echo "== $L"
  RK_LIB=$L timeout 300 python bench.py --workload $WL --no-cpu-baseline --no-extras --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); pk=d['roofline']['per_kernel']
print(round(d['value']), 'fwd', round(pk['forward']['ms'],3), 'bp', round(pk['backproject']['ms'],3))"
  RK_LIB=$L timeout 300 ncu --metrics $M --clock-control none -k regex:${KREGEX:-forward_kernel} -c 1 --csv python tools/prof_step.py $WL 1 32 2>/dev/null | grep -E '"(gpu__|l1tex|smsp|sm__)' | awk -F'","' '{print $(NF-2), $NF}'
done
