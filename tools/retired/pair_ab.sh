#!/bin/bash
# A/B of the parallel backprojector's vertical pixel pairs (RK_BP_PAIR 0/1/2) on the cfg2 bench
# line + the bitwise/parity GPU tests under each mode.  Usage (under gpurun): bash tools/pair_ab.sh
for rep in 1 2; do for M in 0 1 2; do
  RK_BP_PAIR=$M bash tools/ab_bench.sh "paper_2009_14788_b200/libradon_b200.so" "par512" "fp32" 1 | sed "s/^/pair=$M /"
done; done
for M in 1 2; do
  RK_BP_PAIR=$M timeout 600 python -m pytest tests -m gpu -q -x -k "projector or headline or acceptance or solvers" 2>&1 | tail -1 | sed "s/^/pair=$M tests: /"
done
for M in 0 1 2; do
  RK_BP_PAIR=$M timeout 300 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none -k regex:backproject_kernel -c 1 --csv python tools/prof_step.py par512 1 128 2>/dev/null | grep -E '"(gpu__|l1tex|smsp)' | awk -F'","' '{print "pair='$M'", $(NF-2), $NF}'
done
