#!/bin/bash
# A/B of the register tap-reuse variants of the forward / backprojection kernels
# (RK_FWD_REUSE, RK_BP_REUSE), plus GPU parity tests of the default build.
# Usage (under gpurun): bash tools/ab_reuse.sh <tag>
TAG=${1:-ab}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
for cfg in "0 0" "1 0" "2 0" "0 1" "2 1"; do
  set -- $cfg
  RK_FWD_REUSE=$1 RK_BP_REUSE=$2 timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-extras \
    > gpurun_out/bench_${TAG}_f$1b$2.json 2> gpurun_out/bench_${TAG}_f$1b$2.err
  python - "$1" "$2" gpurun_out/bench_${TAG}_f$1b$2.json <<'EOF'
import json, sys
try:
    d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    pk = d["roofline"]["per_kernel"]
    print(f"fwd_reuse={sys.argv[1]} bp_reuse={sys.argv[2]}: {d['value']:.0f} img/s  fwd {pk['forward']['ms']:.3f} ms  bp {pk['backproject']['ms']:.3f} ms")
except Exception as e:
    print("parse failed", sys.argv[1:], e)
EOF
done
# targeted ncu counters of the default (reuse) kernels, batch 32
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:"forward_kernel|backproject_kernel" -c 4 --csv python tools/prof_step.py par512 2 32 > gpurun_out/ncu_counters_$TAG.csv 2> gpurun_out/ncu_counters_$TAG.err
RK_FWD_REUSE=0 RK_BP_REUSE=0 timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:"forward_kernel|backproject_kernel" -c 4 --csv python tools/prof_step.py par512 2 32 > gpurun_out/ncu_counters_${TAG}_plain.csv 2>> gpurun_out/ncu_counters_$TAG.err
