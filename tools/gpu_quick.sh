#!/bin/bash
# Quick GPU A/B: selected GPU tests + par512/fan512 bench lines (fp32, fp16) without side configs.
# Usage (under gpurun): bash tools/gpu_quick.sh <tag> [pytest -k expr]
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x ${2:+-k "$2"} > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -2 gpurun_out/pytest_gpu_$TAG.log
for wl in par512 fan512; do for dt in fp32 fp16; do
  timeout 300 python bench.py --workload $wl --dtype $dt --no-cpu-baseline --no-extras --no-e2e > gpurun_out/bench_${TAG}_${wl}_${dt}.json 2> gpurun_out/bench_${TAG}_${wl}_${dt}.err
  python - gpurun_out/bench_${TAG}_${wl}_${dt}.json $wl $dt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    pk = d["roofline"]["per_kernel"]
    print(f"{sys.argv[2]} {sys.argv[3]}: {d['value']:.0f} img/s  fwd {pk['forward']['ms']:.3f} ms  bp {pk['backproject']['ms']:.3f} ms  frac {d['roofline']['frac']:.3f} parity {d['parity']['max_rel_l2']:.2e} clocks {d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e)
PY
done; done
