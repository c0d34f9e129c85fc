#!/bin/bash
# A/B of the backprojector's thread shape (RK_BP_NARROW: 128 x 8 pixels vs 256 x 4) on the
# cfg2/cfg3 bench lines, the strong-scaling probe and cfg4 FBP.  Usage (under gpurun): bash tools/narrow_ab.sh <tag>
TAG=${1:-nab}
mkdir -p gpurun_out
for rep in 1 2; do for N in 0 1; do
  RK_BP_NARROW=$N bash tools/ab_bench.sh "paper_2009_14788_b200/libradon_b200.so" "par512 fan512" "fp32" 1 | sed "s/^/narrow=$N /"
done; done
for N in 0 1; do
  RK_BP_NARROW=$N timeout 300 python tools/shard_probe.py par512 > gpurun_out/shard_${TAG}_$N.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/shard_${TAG}_$N.json'))
print('narrow=$N shard', {k: (round(v['forward_ms'],3), round(v['backproject_ms'],3), round(v['efficiency_vs_N1'],3)) for k,v in d.items() if k.startswith('N')})"
  RK_BP_NARROW=$N timeout 300 python tools/fbp_probe.py > gpurun_out/fbp_${TAG}_$N.json 2>&1; echo "narrow=$N fbp $(tail -c 300 gpurun_out/fbp_${TAG}_$N.json)"
done
