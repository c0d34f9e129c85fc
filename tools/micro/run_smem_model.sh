#!/bin/bash
# ncu wavefronts per LDS.128 for each lane pattern of smem_model.cu
cd "$(dirname "$0")"
for p in 24 25 26 27 28; do
  ./smem_model $p | head -1
  ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__sass_inst_executed_op_shared_ld.sum --csv ./smem_model $p 2>/dev/null | grep -E "wavefronts|inst_executed" | awk -F'","' '{print $(NF-2), $NF}'
done
