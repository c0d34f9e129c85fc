#!/bin/bash
# Quick GPU check: projector parity tests + a bench line without side configs.
# Usage (under gpurun): bash tools/quick_bench.sh <tag> [pytest -k expr]
TAG=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x ${2:+-k "$2"} > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
RK_DEBUG_PLAN=1 timeout 300 python bench.py --no-cpu-baseline --no-extras > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
grep "\[rk\]" gpurun_out/bench_$TAG.err | head -4
python - gpurun_out/bench_$TAG.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
pk = d["roofline"]["per_kernel"]
print(f"{d['value']:.0f} img/s  e2e {d['e2e']['value']:.0f}  fwd {pk['forward']['ms']:.3f} ms  bp {pk['backproject']['ms']:.3f} ms  frac {d['roofline']['frac']:.3f} clocks {d['clocks']}")
PY
timeout 300 python bench.py --workload fan512 --no-cpu-baseline --no-extras --no-e2e > gpurun_out/bench_${TAG}_fan.json 2> gpurun_out/bench_${TAG}_fan.err
python - gpurun_out/bench_${TAG}_fan.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
pk = d["roofline"]["per_kernel"]
print(f"fan512: {d['value']:.0f} img/s  fwd {pk['forward']['ms']:.3f} ms  bp {pk['backproject']['ms']:.3f} ms")
PY
