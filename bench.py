#!/usr/bin/env python
"""Benchmark: device-timed forward + backprojection images/s on the B200
kernels (BASELINE.json metric, configs[1]: parallel-beam 512x512, 512 angles,
512 detectors, batch 128, fp32), sharded across N GPUs with no collective on
the data path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload par512|fan512|fbp1024]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

One step = forward(images) -> sinogram, then backprojection(sinogram) ->
images, over this rank's contiguous shard of the global batch.  Inputs are
resident in HBM when the timed region starts; the L2 is flushed (a 256 MiB
write) between timed steps, outside the timed events.  Per-kernel device time
comes from the library's own event instrumentation (rk_profiling_*), the
roofline peak from the library's shared-memory bandwidth probe, and the
end-to-end number from the reference-shaped host-buffer entry points
(rk_forward_host / rk_backproject_host: pinned host in, host out, copies in
the timed region).  The CPU baseline is the reference itself compiled in
place (oracle/_ref), timed on this host's cores on a bounded sample.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

# The product package (and so libradon_b200.so) is imported only inside the
# "ours" arm: the --impl reference arm must map nothing but oracle/_ref.

GLOBAL_BATCH = 128
METRIC = "forward+back-projection images/s (512², 512 angles, batch 128) at 1/2/4/8 GPUs"

WORKLOADS = {
    # name: (kind, size, n_angles, angle_stop, det_count, source_distance, global batch)
    "par512": ("parallel", 512, 512, math.pi, 512, 0.0, 128),
    "fan512": ("fanbeam", 512, 512, 2 * math.pi, 512, 512.0, 128),
}


def hbm_check(traffic_bytes, ms):
    """The dominant kernel's measured DRAM traffic (ncu, per launch) over its event-timed duration,
    against the driver-measured HBM copy bandwidth (MEASURED_PEAKS.json)."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if traffic_bytes is None or not os.path.exists(path) or not ms or ms != ms:
        return None
    peak = float(json.load(open(path))["hbm_gbs"])
    gbs = traffic_bytes / (ms * 1e-3) / 1e9
    return {"achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak, "peak_source": "MEASURED_PEAKS.json"}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_images_per_s(wl, budget_s=15.0, warmup=1, fixed_batch=None):
    """The reference (oracle/_ref: radonkit compiled in place) forward + backprojection
    on this host's cores, all threads, on a bounded sample of the workload."""
    from oracle import Geom, RefOracle, default_oracle

    try:
        orc = RefOracle()
        kind = "reference"
    except (FileNotFoundError, OSError):
        orc = default_oracle()
        kind = "port"
    cores = os.cpu_count() or 1
    if kind == "reference":
        orc.set_num_threads(cores)
    k, s, na, stop, nd, src, _ = WORKLOADS[wl]
    g = Geom(k, s, orc.angles_linspace(0.0, stop, na), nd, None, src)
    ph = orc.shepp_logan(s)

    def run(b):
        x = np.repeat(ph, b, axis=0)
        t0 = time.perf_counter()
        y = orc.forward(g, x)
        orc.backprojection(g, y)
        return time.perf_counter() - t0

    t1 = run(1)  # also the warm-up
    for _ in range(max(0, warmup - 1)):
        run(1)
    b = fixed_batch or max(1, min(64, int(budget_s / 5.0 / max(t1, 1e-3))))
    times = [run(b) for _ in range(5)]  # 1 warm-up + >= 5 timed runs, median
    med = statistics.median(times)
    return {"value": b / med, "unit": "images/s", "cores": cores, "kind": kind, **cpu_info(orc),
            "sample": f"{b} x {s}^2 image(s), {na} angles, {nd} cells per run; median of 5 runs after 1 warm-up; "
                      f"{'parallel' if k == 'parallel' else 'fan-beam'}; set_num_threads({cores})"}


def cpu_info(orc):
    """Host CPU model (lscpu 'Model name') and which build of the reference ran (oracle/Makefile)."""
    from oracle import cpu_model

    so = getattr(orc, "path", None)
    return {"cpu_model": cpu_model(), "march": getattr(orc, "march", "x86-64-v3 (port, -O3)"),
            "library": os.path.relpath(so, ROOT) if so else "oracle/_port/liboracle.so"}


def bench_parity(k, s, na, stop, nd, src, imgs, sino, out, tol=1e-5):
    """rel-L2 (tensor.cpp:406-418) of the benched outputs against the reference on the same inputs."""
    from oracle import Geom, default_oracle, rel_l2

    orc = default_oracle()
    if hasattr(orc, "set_num_threads"):
        orc.set_num_threads(os.cpu_count() or 1)
    g = Geom(k, s, orc.angles_linspace(0.0, stop, na), nd, None, src)
    ref_sino = orc.forward(g, imgs)
    ref_bp = orc.backprojection(g, sino)
    fw = [rel_l2(sino[e], ref_sino[e]) for e in range(len(imgs))]
    bp = [rel_l2(out[e], ref_bp[e]) for e in range(len(imgs))]
    return {"max_rel_l2": max(fw + bp), "forward": fw, "backprojection": bp, "tolerance": tol,
            "elements": "0 (phantom x 1/128), 1 (Rng(1) uniform) of the timed batch; bp checked on the GPU sinogram",
            "oracle": os.path.relpath(getattr(orc, "path", "oracle/_port/liboracle.so"), ROOT)}


def reference_cfg5(args, orc, kind, cores):
    """--impl reference --workload cfg5: the reference's landweber (solvers.cpp:130-145), 50
    iterations, one image of the config-5 batch per step (the bounded sample)."""
    from oracle import Geom

    g = Geom("parallel", 512, orc.angles_linspace(0.0, math.pi, 256))
    x = orc.shepp_logan(512) * np.float32(1.0 / 256.0)
    y = orc.forward(g, x)
    alpha = 0.95 * orc.estimate_alpha(g, 20, 0) if hasattr(orc, "estimate_alpha") else 1e-5
    times = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        orc.landweber(g, y, np.zeros_like(x), alpha, 50)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = args.steps / tot
    line = {
        "impl": "reference", "metric": "reconstructed images/s (50 Landweber iterations, 512^2, 256 angles, batch 256)",
        "value": value, "unit": "images/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": 0,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "fp32 state, fp64 accumulate", "data": "synthetic: shepp_logan(512) / 256",
        "config": {"workload": "cfg5: parallel 512x512, linspace(0, pi, 256), 512 cells, global batch 256, "
                               "50 iterations", "sample_per_step": 1},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": kind, **cpu_info(orc),
                         "sample": "1 image x 50 Landweber iterations per step"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_reference_arm(args):
    """--impl reference: the reference's own CPU implementation on the host cores."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    from oracle import Geom, RefOracle, default_oracle

    try:
        orc = RefOracle()
        kind = "reference"
    except (FileNotFoundError, OSError):
        orc = default_oracle()
        kind = "port"
    cores = os.cpu_count() or 1
    if kind == "reference":
        orc.set_num_threads(cores)
    if args.workload == "cfg5":
        return reference_cfg5(args, orc, kind, cores)
    k, s, na, stop, nd, src, B = WORKLOADS[args.workload]
    g = Geom(k, s, orc.angles_linspace(0.0, stop, na), nd, None, src)
    ph = orc.shepp_logan(s)
    x1 = ph.copy()
    t0 = time.perf_counter()
    orc.backprojection(g, orc.forward(g, x1))
    t1 = time.perf_counter() - t0
    per_step = max(1, min(B, int(6.0 / max(t1, 1e-3))))  # bounded sample: ~6 s of CPU work per step
    x = np.repeat(ph, per_step, axis=0)
    for _ in range(args.warmup):
        orc.backprojection(g, orc.forward(g, x[:1]))
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        orc.backprojection(g, orc.forward(g, x))
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = per_step * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32 storage, fp64 accumulate",
        "data": "synthetic: modified Shepp-Logan phantom (reference shepp_logan)",
        "config": {"workload": f"{args.workload}: {k} {s}x{s}, {na} angles, {nd} detectors, global batch {B}",
                   "sample_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": kind, **cpu_info(orc),
                         "sample": f"{per_step} image(s) per step of the {args.workload} workload"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="par512", choices=sorted(WORKLOADS) + ["cfg5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "fp16"],
                    help="storage dtype of images and sinograms (fp32 compute either way; projector.cpp:207-224)")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of the timed outputs")
    ap.add_argument("--no-extras", action="store_true", help="skip the config 3/4/5 side measurements")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch

    import paper_2009_14788_b200 as rk
    from paper_2009_14788_b200 import _lib
    from paper_2009_14788_b200.phantom import shepp_logan as rk_phantom  # synthetic input

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    # RK_BENCH_SHARE_DEVICE=1: every rank on cuda:0 — exercises the multi-rank path (init,
    # barriers, max-over-ranks, sharding) on a one-GPU box; NCCL rejects two ranks on one
    # device, so that mode defaults to gloo (RK_BENCH_BACKEND overrides either default).
    share = os.environ.get("RK_BENCH_SHARE_DEVICE", "0") == "1"
    gpu = 0 if share else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    dist = None
    backend = os.environ.get("RK_BENCH_BACKEND", "gloo" if share else "nccl")
    # RK_BENCH_FORCE_DIST=1: initialise the process group even at world size 1, so a one-GPU box
    # runs the real NCCL init / barrier / max-reduce lines (NCCL rejects two ranks on one device)
    if world > 1 or os.environ.get("RK_BENCH_FORCE_DIST", "0") == "1":
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def max_over_ranks(v):
        """Device-timed value -> max over ranks (the contract's multi-GPU time)."""
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if args.workload == "cfg5":
        return run_cfg5(args, rk, _lib, torch, dist, dev, gpu, world, rank, backend, max_over_ranks)

    k, s, na, stop, nd, src, B = WORKLOADS[args.workload]
    ang = rk.angles_linspace(0.0, stop, na)
    g = rk.make_parallel(s, ang, nd) if k == "parallel" else rk.make_fanbeam(s, ang, src, det_count=nd)
    from paper_2009_14788_b200.sharding import shard_range

    lo, hi = shard_range(B, world, rank)  # contiguous batch shard, no data-path collective
    nb = hi - lo

    # synthetic inputs: phantom x (e+1)/128, Rng(seed=e) uniform for odd e
    ph = rk_phantom(s)
    imgs = np.empty((nb, s, s), np.float32)
    for i, e in enumerate(range(lo, hi)):
        if e % 2 == 0:
            imgs[i] = ph * np.float32((e + 1) / 128.0)
        else:
            imgs[i] = rk.Rng(e).uniform_tensor((s, s))
    fp16 = args.dtype == "fp16"
    tdt = torch.float16 if fp16 else torch.float32
    rkdt = _lib.RK_F16 if fp16 else _lib.RK_F32
    esz = 2 if fp16 else 4
    if fp16:  # x 1/8: the backprojection of a 512-angle sinogram stays inside the half range (65504)
        imgs = (imgs * np.float32(0.125)).astype(np.float16)
    x = torch.from_numpy(imgs).to(dev)
    sino = torch.empty(nb, na, nd, device=dev, dtype=tdt)
    out = torch.empty(nb, s, s, device=dev, dtype=tdt)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    plan = rk.get_plan(g, None, gpu)
    info = plan.info()
    stream = torch.cuda.current_stream(dev)
    sp = ctypes_void(stream.cuda_stream)

    def step():
        _lib.check(_lib.lib.rk_forward(plan.handle, rkdt, ctypes_void(x.data_ptr()), nb,
                                       ctypes_void(sino.data_ptr()), sp))
        _lib.check(_lib.lib.rk_backproject(plan.handle, rkdt, ctypes_void(sino.data_ptr()), nb,
                                           ctypes_void(out.data_ptr()), sp))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    smem_peak = ctypes_double()
    _lib.check(_lib.lib.rk_probe_smem_bandwidth(gpu, smem_peak))
    stats = _lib.RkKernelStats()
    _lib.check(_lib.lib.rk_profiling_read(ctypes_ref(stats), 1))

    # a timed region that saw a hardware / thermal slowdown is measured once more (the
    # contract rejects such a run); the decision is collective so every rank repeats it
    remeasured = False
    for attempt in range(2):
        clocks = ClockSampler(gpu)
        clocks.start()
        time.sleep(0.3)
        _lib.check(_lib.lib.rk_profiling_read(ctypes_ref(stats), 1))  # reset the per-kind counters
        _lib.check(_lib.lib.rk_profiling_enable(1))
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # L2 flush between timed steps (outside the events)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        _lib.check(_lib.lib.rk_profiling_enable(0))
        _lib.check(_lib.lib.rk_profiling_read(ctypes_ref(stats), 1))
        clk = clocks.stop()
        bad = bool(set(clk.get("reasons", [])) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"})
        if attempt == 1 or max_over_ranks(1.0 if bad else 0.0) == 0.0:
            break
        remeasured = True
    clk["remeasured"] = remeasured
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = max_over_ranks(sum(step_ms))
    ms_per_step = total_ms / args.steps
    value = B / (ms_per_step * 1e-3)

    kinds = _lib.KERNEL_KINDS
    launches = int(sum(stats.launches[i] for i in range(len(kinds))))
    kern = {kinds[i]: {"launches": int(stats.launches[i]), "ms_total": float(stats.ms[i]),
                       "ms_per_launch": (float(stats.ms[i]) / stats.timed[i]) if stats.timed[i] else None}
            for i in range(len(kinds)) if stats.launches[i]}
    # roofline of the dominant kernel: algorithmic L1TEX/SMEM bytes per launch
    # (16 B per forward sample = 4 fp32 taps; 8 B per backprojection sample = 2 taps)
    # fp16 storage: 4 taps x 2 B forward, 2 taps x 2 B backprojection
    fwd_bps, bp_bps = (8, 4) if fp16 else (16, 8)
    fwd_bytes = float(fwd_bps) * info["forward_samples"] * nb
    bp_bytes = float(bp_bps) * info["backproject_samples"] * nb
    fwd_ms = kern.get("forward", {}).get("ms_per_launch") or float("nan")
    bp_ms = kern.get("backproject", {}).get("ms_per_launch") or float("nan")
    dom, dbytes, dms = ("forward", fwd_bytes, fwd_ms) if fwd_ms >= bp_ms else ("backproject", bp_bytes, bp_ms)
    achieved = dbytes / (dms * 1e-3) / 1e9
    peak = float(smem_peak.value)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        rec = json.load(open(tfile)).get(args.workload, {}).get(dom)
        if rec:  # DRAM bytes per launch from the committed ncu --set full capture, rescaled to this batch
            traffic = rec["bytes_per_image"] * nb
    roofline = {"bound": "l1tex", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch (profiles/ncu_traffic.json); "
                                "HBM is not the binding resource: the kernel's data path is shared memory",
                "peak_source": "measured in this run by rk_probe_smem_bandwidth (LDS.128, all SMs); "
                               "MEASURED_PEAKS.json has no L1TEX/SMEM figure",
                "peak_nominal": 148 * 128 * 1.965,  # SMs x 128 B/clk (one LDS wavefront) x max SM clock, GB/s
                "bound_note": "neither HBM nor the tensor cores bind this gather kernel (SURVEY 8d): its "
                              "algorithmic unit is the shared-memory tap read, so the peak is the L1TEX/SMEM "
                              "bandwidth; the HBM check below uses MEASURED_PEAKS.json",
                "hbm_check": hbm_check(traffic, dms),
                "algorithmic_bytes_per_launch": dbytes,
                "per_kernel": {
                    "forward": {"samples_per_launch": info["forward_samples"] * nb, "bytes_per_sample": fwd_bps,
                                "ms": fwd_ms, "gbs": fwd_bytes / (fwd_ms * 1e-3) / 1e9,
                                "gsamples_per_s": info["forward_samples"] * nb / (fwd_ms * 1e-3) / 1e9},
                    "backproject": {"samples_per_launch": info["backproject_samples"] * nb, "bytes_per_sample": bp_bps,
                                    "ms": bp_ms, "gbs": bp_bytes / (bp_ms * 1e-3) / 1e9,
                                    "gsamples_per_s": info["backproject_samples"] * nb / (bp_ms * 1e-3) / 1e9}}}

    # ---- parity of the timed step's own outputs (checker only, outside every timed region):
    # rel-L2 of elements 0-1 of this rank's shard against the reference (oracle/_ref) on the
    # benched geometry: forward on the input images, backprojection on the GPU's sinogram.
    parity = None
    if rank == 0 and not args.no_parity:
        parity = bench_parity(k, s, na, stop, nd, src, imgs[:2], sino[:2].cpu().numpy(), out[:2].cpu().numpy(),
                              1e-3 if fp16 else 1e-5)

    # ---- end to end through the reference-shaped host-buffer API
    e2e = None
    if not args.no_e2e:
        h_img = torch.from_numpy(imgs).pin_memory()
        h_sino = torch.empty(nb, na, nd, dtype=tdt).pin_memory()
        h_out = torch.empty(nb, s, s, dtype=tdt).pin_memory()

        def e2e_step():
            _lib.check(_lib.lib.rk_forward_host(plan.handle, rkdt, ctypes_void(h_img.data_ptr()), nb,
                                                ctypes_void(h_sino.data_ptr())))
            _lib.check(_lib.lib.rk_backproject_host(plan.handle, rkdt, ctypes_void(h_sino.data_ptr()), nb,
                                                    ctypes_void(h_out.data_ptr())))

        for _ in range(2):
            e2e_step()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        el = max_over_ranks(time.perf_counter() - t0)
        bi = esz * nb * (s * s + na * nd)
        e2e = {"value": B * args.steps / el, "unit": "images/s", "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bi,
               "ms_per_step": 1e3 * el / args.steps,
               "path": "rk_forward_host + rk_backproject_host (pinned host buffers, 3-stream chunked copy/compute "
                       "pipeline, synchronous like the reference's Tensor-in/Tensor-out calls)"}

    if e2e is not None and rank == 0:
        e2e["first_call_ms"] = first_call_latency(rk, _lib, g, gpu, np.ascontiguousarray(imgs[:1], np.float32))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference_images_per_s(args.workload)
    extras = None
    if world == 1 and not args.no_extras:
        del x, sino, out, flush
        torch.cuda.empty_cache()
        extras = measure_extras(rk, _lib, dev)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp16 storage, fp32 compute" if fp16 else "fp32",
            "data": "synthetic: modified Shepp-Logan phantom x (e+1)/128 for even e, Rng(e) uniform for odd e"
                    + (", x 1/8 in fp16 storage" if fp16 else ""),
            "config": {"workload": f"{args.workload}: {k} {s}x{s}, {na} angles, {nd} detectors, global batch {B}",
                       "global_batch": B, "per_gpu_batch": nb, "parallelism": f"batch-shard x{world}, no collective",
                       "dist_backend": backend if dist is not None else None, "shared_device": share,
                       "l2": "flushed (256 MiB write) between timed steps, outside the timed events"},
            "roofline": roofline, "parity": parity, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "kernels": kern,
            "clocks": clk, "other_configs": extras,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def first_call_latency(rk, _lib, g, gpu, img1, reps=3):
    """One-shot latency of the reference-shaped call (projector.cpp:228-236: a stateless forward):
    a new plan + the first rk_forward_host of one image (host buffers, copies included), with the
    forward schedule planned from scratch ("cold": empty plan cache), read from the on-disk plan
    cache ("warm_cache": a new process projecting a geometry seen before), and a second call on the
    same plan ("steady").  Median of `reps` rounds, each with a fresh cache directory."""
    import tempfile

    from paper_2009_14788_b200.projector import Plan

    na, nd = g.n_angles, g.det_count
    out = np.empty((1, na, nd), np.float32)
    saved = os.environ.get("RK_PLAN_CACHE")
    runs = {"cold": [], "warm_cache": [], "steady": []}
    try:
        for _ in range(reps):
            os.environ["RK_PLAN_CACHE"] = tempfile.mkdtemp(prefix="rk_bench_cache_")
            for key in ("cold", "warm_cache"):
                t0 = time.perf_counter()
                p = Plan(g, 1.0, gpu)
                _lib.check(_lib.lib.rk_forward_host(p.handle, _lib.RK_F32, ctypes_void(img1.ctypes.data), 1,
                                                    ctypes_void(out.ctypes.data)))
                runs[key].append(1e3 * (time.perf_counter() - t0))
                assert p.info()["schedule_from_cache"] == (key == "warm_cache")
                if key == "warm_cache":
                    t0 = time.perf_counter()
                    _lib.check(_lib.lib.rk_forward_host(p.handle, _lib.RK_F32, ctypes_void(img1.ctypes.data), 1,
                                                        ctypes_void(out.ctypes.data)))
                    runs["steady"].append(1e3 * (time.perf_counter() - t0))
                del p
    finally:
        if saved is None:
            os.environ.pop("RK_PLAN_CACHE", None)
        else:
            os.environ["RK_PLAN_CACHE"] = saved
    res = {k: statistics.median(v) for k, v in runs.items()}
    res["runs"] = {k: [round(x, 2) for x in v] for k, v in runs.items()}
    res["what"] = ("new plan + first rk_forward_host of 1 image (pageable host buffers): schedule planned (cold), "
                   "read from the plan cache (warm_cache); steady = the next call on the same plan; median of "
                   f"{reps} rounds (fresh cache directory each)")
    return res


def run_cfg5(args, rk, _lib, torch, dist, dev, gpu, world, rank, backend, max_over_ranks):
    """--workload cfg5 (BASELINE configs[4]): 50 Landweber iterations
    (solvers.cpp:130-145, alpha = 0.95 estimate_alpha(op, 20, seed 0)) on parallel 512^2,
    linspace(0, pi, 256), 512 cells, global batch 256 sharded over the ranks with no collective;
    50 CGNE iterations (solvers.cpp:147-166) measured beside it.  A step = one solve of this
    rank's shard; device time by CUDA events, max over ranks."""
    from paper_2009_14788_b200.phantom import shepp_logan
    from paper_2009_14788_b200.sharding import shard_range

    B, iters = 256, 50
    g = rk.make_parallel(512, rk.angles_linspace(0.0, math.pi, 256))
    op = rk.projector_operator(g)
    lo, hi = shard_range(B, world, rank)
    nb = hi - lo
    ph = shepp_logan(512)
    x = torch.from_numpy(np.stack([ph * np.float32((e + 1) / float(B)) for e in range(lo, hi)])).to(dev)
    y = rk.forward(g, x)
    z = torch.zeros_like(x)
    alpha = 0.95 * rk.estimate_alpha(op, 20, 0)  # deterministic: every rank derives the same step
    st = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def timed(fn, steps):
        tot = 0.0
        for i in range(steps):
            flush.fill_(i & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            torch.cuda.synchronize(dev)
            tot += a.elapsed_time(b)
        return tot

    lw = lambda: rk.landweber(op, y, z, alpha, iters)  # noqa: E731
    cg = lambda: rk.cgne(op, z, y, iters)  # noqa: E731
    for _ in range(args.warmup):
        lw()
    cg()
    torch.cuda.synchronize(dev)
    stats = _lib.RkKernelStats()
    _lib.check(_lib.lib.rk_profiling_read(ctypes_ref(stats), 1))
    clocks = ClockSampler(gpu)
    clocks.start()
    time.sleep(0.3)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ms_lw = max_over_ranks(timed(lw, args.steps))
    _lib.check(_lib.lib.rk_profiling_read(ctypes_ref(stats), 1))
    launches = int(sum(stats.launches[i] for i in range(len(_lib.KERNEL_KINDS))))
    ms_cg = max_over_ranks(timed(cg, max(1, args.steps // 2)))
    clk = clocks.stop()
    if dist is not None:
        dist.barrier()
    per_lw = ms_lw / args.steps
    per_cg = ms_cg / max(1, args.steps // 2)
    if rank == 0:
        line = {
            "metric": "reconstructed images/s (50 Landweber iterations, 512^2, 256 angles, batch 256)",
            "value": B / (per_lw * 1e-3), "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_lw, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic: shepp_logan(512) x (e+1)/256",
            "config": {"workload": "cfg5: parallel 512x512, linspace(0, pi, 256), 512 cells, global batch 256, "
                                   "50 iterations", "global_batch": B, "per_gpu_batch": nb,
                       "parallelism": f"batch-shard x{world}, no collective",
                       "dist_backend": backend if dist is not None else None, "alpha": alpha,
                       "alpha_note": "0.95 * estimate_alpha(op, 20, seed 0), computed once outside the timed region",
                       "l2": "flushed (256 MiB write) between timed steps, outside the timed events"},
            "cgne": {"value": B / (per_cg * 1e-3), "unit": "images/s", "ms_per_step": per_cg,
                     "steps": max(1, args.steps // 2)},
            "gpu_launches": launches, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def measure_extras(rk, _lib, dev):
    """Device-timed numbers for the other BASELINE configs (N=1 only; 1 warm-up + 3 runs each)."""
    import torch

    from paper_2009_14788_b200.phantom import shepp_logan as rk_phantom  # synthetic input

    out = {}
    st = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def timed(fn, runs=3):
        fn()
        torch.cuda.synchronize(dev)
        tot = 0.0
        for i in range(runs):
            flush.fill_(i)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            torch.cuda.synchronize(dev)
            tot += a.elapsed_time(b)
        return tot / runs

    # config 3: fan-beam 512^2, 512 angles over 2 pi, D_so = D_dd = 512, batch 128, fp32
    gf = rk.make_fanbeam(512, rk.angles_linspace(0.0, 2 * math.pi, 512), 512.0)
    x = torch.from_numpy(np.stack([rk_phantom(512) * ((e + 1) / 128.0) for e in range(128)])).to(dev)
    y = rk.forward(gf, x)
    ms = timed(lambda: rk.backprojection(gf, rk.forward(gf, x)))
    out["cfg3_fan512_b128_fp32"] = {"metric": "forward+backprojection images/s", "value": 128 / (ms * 1e-3),
                                    "ms": ms}
    # the same through the host-buffer entry points (pinned buffers, copies inside), wall clock
    pf = rk.get_plan(gf, None, dev.index or 0)
    h_img = x.cpu().pin_memory()
    h_sino, h_out = torch.empty(tuple(y.shape)).pin_memory(), torch.empty(tuple(x.shape)).pin_memory()

    def host_pair():
        _lib.check(_lib.lib.rk_forward_host(pf.handle, _lib.RK_F32, ctypes_void(h_img.data_ptr()), 128,
                                            ctypes_void(h_sino.data_ptr())))
        _lib.check(_lib.lib.rk_backproject_host(pf.handle, _lib.RK_F32, ctypes_void(h_sino.data_ptr()), 128,
                                                ctypes_void(h_out.data_ptr())))

    host_pair()
    t0 = time.perf_counter()
    for _ in range(3):
        host_pair()
    el = (time.perf_counter() - t0) / 3
    out["cfg3_fan512_b128_fp32"]["e2e"] = {"value": 128 / el, "unit": "images/s", "ms": 1e3 * el,
                                           "h2d_bytes_per_step": h_img.numel() * 4 + h_sino.numel() * 4,
                                           "d2h_bytes_per_step": h_sino.numel() * 4 + h_out.numel() * 4}
    del x, y, h_img, h_sino, h_out
    # config 4: FBP 1024^2, 720 angles, nd 1024 and 1449, batch 64, fp32 and fp16 storage
    ph = rk_phantom(1024)
    x = torch.from_numpy(np.stack([ph * ((e + 1) / 64.0) for e in range(64)])).to(dev)
    for nd in (1024, 1449):
        g4 = rk.make_parallel(1024, rk.angles_linspace(0.0, math.pi, 720), nd)
        sino = rk.forward(g4, x)
        for dt, name in ((torch.float32, "fp32"), (torch.float16, "fp16")):
            s_ = sino.to(dt)
            ms = timed(lambda: rk.fbp(g4, s_))
            out[f"cfg4_fbp1024_720_nd{nd}_b64_{name}"] = {"metric": "FBP images/s", "value": 64 / (ms * 1e-3), "ms": ms}
        del sino
    del x
    # config 5: 50 Landweber / CGNE iterations, 512^2, 256 angles, batch 256 (the whole 8-GPU batch on one GPU)
    g5 = rk.make_parallel(512, rk.angles_linspace(0.0, math.pi, 256))
    op = rk.projector_operator(g5)
    x = torch.from_numpy(np.stack([rk_phantom(512) * ((e + 1) / 256.0) for e in range(256)])).to(dev)
    y = rk.forward(g5, x)
    z = torch.zeros_like(x)
    alpha = 0.95 * rk.estimate_alpha(op, 20, 0)
    ms = timed(lambda: rk.landweber(op, y, z, alpha, 50), runs=1)
    out["cfg5_landweber50_512_256_b256"] = {"metric": "reconstructed images/s (50 iterations)",
                                            "value": 256 / (ms * 1e-3), "ms": ms, "alpha": alpha}
    ms = timed(lambda: rk.cgne(op, z, y, 50), runs=1)
    out["cfg5_cgne50_512_256_b256"] = {"metric": "reconstructed images/s (50 iterations)", "value": 256 / (ms * 1e-3),
                                       "ms": ms}
    del x, y, z
    # alpha-shearlet analysis / synthesis, 512^2, 5 scales at alpha 0.5 (59 coefficients), batch 8
    plan = rk.make_plan(512, 512, [0.5] * 5)
    x = torch.from_numpy(np.stack([rk_phantom(512) * ((e + 1) / 8.0) for e in range(8)])).to(dev)
    c = rk.forward(plan, x)
    ms_f = timed(lambda: rk.forward(plan, x))
    ms_b = timed(lambda: rk.backward(plan, c))
    out["next_shearlet512_s5_b8_fp32"] = {"metric": "shearlet analysis / synthesis images/s", "forward": 8 / (ms_f * 1e-3),
                                          "backward": 8 / (ms_b * 1e-3), "ms_forward": ms_f, "ms_backward": ms_b,
                                          "n_coeff": plan.n_coeff}
    del c
    # the paper's ADMM: 512^2, limited 100 degree arc, 512 angles,
    # 5 scales, p0 0.02, p1 0.1, 50 outer x 50 inner iterations; batch 1 and 8
    ga = rk.make_parallel(512, [(i * 100.0 / 512 - 50.0) * math.pi / 180.0 for i in range(512)])
    opa = rk.projector_operator(ga)
    for b in (1, 8):
        ya = rk.forward(ga, x[:b])
        # warm-up: plans, scratch and GPU clocks (a short run leaves the clocks ramping into the timed one)
        rk.admm_reconstruct(opa, plan, ya, rk.AdmmParams(outer_iterations=20, inner_cg_iterations=50))
        # median of three full calls: single runs on a shared box showed +25-50 % outliers
        # (tools/admm_var_probe.py: per-iteration device time is flat at 19.0 ms for batch 1)
        runs = []
        for _ in range(3):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            a.record(st)
            rk.admm_reconstruct(opa, plan, ya, rk.AdmmParams(outer_iterations=50, inner_cg_iterations=50))
            e.record(st)
            torch.cuda.synchronize(dev)
            runs.append(a.elapsed_time(e))
        runs.sort()
        ms = runs[1]
        out[f"next_admm512_limited100_na512_b{b}_fp32"] = {"metric": "ADMM seconds per image (50 outer x 50 inner)",
                                                           "value": ms * 1e-3 / b, "ms": ms,
                                                           "runs_ms": [round(r, 1) for r in runs],
                                                           "paper_v100_s_per_image": 1.6 if b == 1 else 1.2}
    return out


def ctypes_void(p):
    import ctypes

    return ctypes.c_void_p(p)


def ctypes_double():
    import ctypes

    return ctypes.c_double()


def ctypes_ref(x):
    import ctypes

    return ctypes.byref(x)


if __name__ == "__main__":
    sys.exit(main())
