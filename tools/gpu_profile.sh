#!/bin/bash
# Round profile pass (one GPU): GPU suite, smoke, bench + reference arm, the
# multi-rank path on one GPU, the bench launch list and ncu --set full
# captures of the projector kernels (fp32 par/fan, fp16 par) and the filter.
# Usage (under gpurun): bash tools/gpu_profile.sh <tag> [skip-tests]
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -rA --durations=10 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
  grep -E "passed|failed|FAILED|ERROR" gpurun_out/pytest_gpu_$TAG.log | tail -8
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 300 gpurun_out/bench_$TAG.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1; tail -c 200 gpurun_out/bench_ref_$TAG.json; echo
for dt in fp16; do for wl in par512 fan512; do
  timeout 300 python bench.py --workload $wl --dtype $dt --no-cpu-baseline --no-extras > gpurun_out/bench_${TAG}_${wl}_${dt}.json 2>/dev/null
done; done
RK_BENCH_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --no-extras > gpurun_out/bench_tr2_gloo_$TAG.json 2> gpurun_out/bench_tr2_gloo_$TAG.err; echo "tr2 gloo rc=$?"
RK_BENCH_FORCE_DIST=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_tr1_nccl_$TAG.json 2> gpurun_out/bench_tr1_nccl_$TAG.err; echo "tr1 nccl rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-extras --no-parity > gpurun_out/launches_$TAG.stdout 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"forward_kernel|backproject_kernel" -s 2 -c 2 -o gpurun_out/prof_${TAG}_par python tools/prof_step.py par512 2 128 > gpurun_out/ncu_${TAG}_par.log 2>&1; tail -1 gpurun_out/ncu_${TAG}_par.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"forward_kernel|backproject_kernel" -s 2 -c 2 -o gpurun_out/prof_${TAG}_fan python tools/prof_step.py fan512 2 128 > gpurun_out/ncu_${TAG}_fan.log 2>&1; tail -1 gpurun_out/ncu_${TAG}_fan.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"forward_kernel|backproject_kernel" -s 2 -c 2 -o gpurun_out/prof_${TAG}_h8 python tools/prof_step.py par512 2 128 f16 > gpurun_out/ncu_${TAG}_h8.log 2>&1; tail -1 gpurun_out/ncu_${TAG}_h8.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"filter_kernel" -s 1 -c 1 -o gpurun_out/prof_${TAG}_filter python tools/prof_fbp.py 1024 2 > gpurun_out/ncu_${TAG}_filter.log 2>&1; tail -1 gpurun_out/ncu_${TAG}_filter.log
timeout 600 python tools/shard_probe.py par512 > gpurun_out/shard_probe_${TAG}_par.json 2>&1; tail -c 400 gpurun_out/shard_probe_${TAG}_par.json; echo
timeout 600 python tools/b1_probe.py > gpurun_out/b1_probe_${TAG}.json 2>&1; tail -c 300 gpurun_out/b1_probe_${TAG}.json; echo
timeout 600 python tools/fbp_probe.py > gpurun_out/fbp_probe_${TAG}.json 2>&1; tail -c 300 gpurun_out/fbp_probe_${TAG}.json; echo
# summarise the captures on the box and drop the reports (gpurun copies back <= 64 MiB)
for t in par fan h8 filter; do
  if [ -f gpurun_out/prof_${TAG}_$t.ncu-rep ]; then
    python tools/ncu_summary.py gpurun_out/prof_${TAG}_$t.ncu-rep $( [ $t = par ] && echo gpurun_out/launches_$TAG.csv ) > gpurun_out/ncu_summary_${TAG}_$t.md 2>&1
    [ "${KEEP_REPS:-0}" = 1 ] || rm -f gpurun_out/prof_${TAG}_$t.ncu-rep
  fi
done
