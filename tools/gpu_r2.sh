#!/bin/bash
# Round-2 GPU session: full GPU suite, smoke, bench (ours + reference arm), the
# multi-rank path on one GPU (torchrun x2, shared device), sharded cfg5.
# Usage (under gpurun): bash tools/gpu_r2.sh <tag> [skip-tests]
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
lscpu > gpurun_out/lscpu_$TAG.txt 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -rA --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
  grep -E "passed|failed|FAILED|ERROR" gpurun_out/pytest_gpu_$TAG.log | tail -15
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -2 gpurun_out/smoke_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 400 gpurun_out/bench_$TAG.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1; tail -c 300 gpurun_out/bench_ref_$TAG.json; echo
RK_BENCH_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_tr2_gloo_$TAG.json 2> gpurun_out/bench_tr2_gloo_$TAG.err; echo "tr2 gloo rc=$?"; tail -c 300 gpurun_out/bench_tr2_gloo_$TAG.json; echo
RK_BENCH_FORCE_DIST=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_tr1_nccl_$TAG.json 2> gpurun_out/bench_tr1_nccl_$TAG.err; echo "tr1 nccl rc=$?"; tail -c 300 gpurun_out/bench_tr1_nccl_$TAG.json; echo
timeout 600 python bench.py --workload cfg5 --steps 4 > gpurun_out/bench_cfg5_$TAG.json 2> gpurun_out/bench_cfg5_$TAG.err; tail -c 300 gpurun_out/bench_cfg5_$TAG.json; echo
RK_BENCH_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --workload cfg5 --steps 2 > gpurun_out/bench_cfg5_tr2_$TAG.json 2> gpurun_out/bench_cfg5_tr2_$TAG.err; echo "cfg5 tr2 rc=$?"; tail -c 300 gpurun_out/bench_cfg5_tr2_$TAG.json; echo
