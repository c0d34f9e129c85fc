"""Randomised parity sweep (GPU vs the reference compiled in place): many more geometries,
batch sizes (all kernel variants: single-lane, WIDE, 128 x 8, half8) and storage dtypes than
the committed test suite.  Prints one line per failure and a summary; exit 1 on any failure.

  python tools/stress_parity.py [n_cases] [seed] [max_size]
"""
import dataclasses
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402
from oracle import Geom, default_oracle, rel_l2  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
only = set(int(v) for v in os.environ.get("RK_STRESS_ONLY", "").split(",") if v)  # replay chosen case indices
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
max_size = int(sys.argv[3]) if len(sys.argv) > 3 else 260
orc = default_oracle()
rs = np.random.default_rng(seed)
fails, worst, t0, ran = 0, {"fp32": (0.0, ""), "fp16": (0.0, ""), "fp64": (0.0, "")}, time.time(), 0
for c in range(n_cases):
    s = int(rs.choice([1, 2, 3, 5, 8, 17, 31, 32, 33, 64, 65, 96, 100, 128, 129, int(rs.integers(4, max_size))]))
    kind = "fan" if rs.random() < 0.45 else "par"
    na = int(rs.choice([1, 2, 7, 30, 64, int(rs.integers(1, 200))]))
    if rs.random() < 0.5:
        ang = list(np.linspace(0.0, (2 * np.pi if kind == "fan" else np.pi), na, endpoint=False))
    else:
        ang = list(rs.uniform(-7.0, 7.0, na))
    nd = int(rs.integers(1, 2 * s + 8)) if rs.random() < 0.5 else None
    sp = float(rs.uniform(0.4, 2.5)) if rs.random() < 0.5 else None
    try:
        if kind == "par":
            g = rk.make_parallel(s, ang, nd, sp)
        else:
            src = float(s) * float(rs.uniform(0.75, 4.0))
            g = rk.make_fanbeam(s, ang, src, float(rs.uniform(0.5, 3.0)) * s if rs.random() < 0.5 else None, nd, sp)
    except rk.ValidationError:
        continue
    ran += 1
    og = (Geom("fanbeam", s, np.asarray(g.angles), g.det_count, g.det_spacing, g.source_distance, g.det_distance)
          if kind == "fan" else Geom("parallel", s, np.asarray(g.angles), g.det_count, g.det_spacing))
    B = int(rs.choice([1, 2, 3, 4, 5, 8, 9, 12, 13, 16, 17]))
    u = rs.random()
    dt = "fp16" if u < 0.25 else ("fp64" if u < 0.35 else "fp32")
    npdt, tdt, tol = {"fp16": (np.float16, torch.float16, 1e-3), "fp32": (np.float32, torch.float32, 1e-5),
                      "fp64": (np.float64, torch.float64, 1e-5)}[dt]
    step = float(rs.choice([1.0, 1.0, 1.0, 0.5, 1.7]))
    host_path = rs.random() < 0.2  # numpy in/out: the *_host entry points
    filt = str(rs.choice(["ram-lak", "shepp-logan", "cosine", "hamming", "hann"])) if rs.random() < 0.3 else None
    x = (rs.uniform(0.0, 1.0, (B, s, s)) * (0.25 if dt == "fp16" else 1.0)).astype(npdt)
    y = (rs.standard_normal((B, g.n_angles, g.det_count)) * (0.05 if dt == "fp16" else 1.0)).astype(npdt)
    if only and c not in only:
        continue
    if only:
        print(f"case {c}: {kind} s={s} angles={list(g.angles)[:4]} nd={g.det_count} sp={g.det_spacing!r} "
              f"src={getattr(g, 'source_distance', None)} dd={getattr(g, 'det_distance', None)} B={B} {dt}")
    try:
        opts = rk.ProjectorOptions(step)
        if host_path:
            f = np.asarray(rk.forward(g, x, opts))
            b = np.asarray(rk.backprojection(g, y))
        else:
            f = rk.forward(g, torch.from_numpy(x).cuda(), opts).cpu().numpy()
            b = rk.backprojection(g, torch.from_numpy(y).cuda()).cpu().numpy()
        fb = None
        if filt is not None and g.det_count < 2:  # make_filter rejects it, as the reference (sino_filter.cpp:65)
            try:
                rk.fbp(g, y if host_path else torch.from_numpy(y).cuda(), rk.filter_kind_from_name(filt))
                raise AssertionError("fbp accepted det_count < 2")
            except rk.ValidationError as ve:
                assert "det_count must be >= 2" in str(ve), ve
            filt = None
        if filt is not None and dt != "fp64":
            yin = y if host_path else torch.from_numpy(y).cuda()
            fb = rk.fbp(g, yin, rk.filter_kind_from_name(filt))
            fb = np.asarray(fb) if host_path else fb.cpu().numpy()
    except Exception as exc:  # noqa: BLE001 — a geometry the library rejects is a failure here
        fails += 1
        print(f"FAIL case {c}: {kind} s={s} na={g.n_angles} nd={g.det_count} sp={g.det_spacing!r} "
              f"src={getattr(g, 'source_distance', None)} dd={getattr(g, 'det_distance', None)} angles[:3]="
              f"{list(g.angles)[:3]} B={B}: {exc}", flush=True)
        continue
    og_step = dataclasses.replace(og, step=step)
    rf, rb = orc.forward(og_step, x), orc.backprojection(og, y)
    checks = [("forward", f, rf), ("backprojection", b, rb)]
    if fb is not None:
        checks.append((f"fbp-{filt}", fb, orc.fbp(og, y, filt)))
    for name, a, r in checks:
        a32, r32 = a.astype(np.float64), r.astype(np.float64)
        if not np.isfinite(r32).all():
            continue  # fp16 overflow cases are tested separately
        if np.abs(r32).max() == 0:
            ok, e = np.abs(a32).max() == 0, 0.0
        else:
            e = rel_l2(a32, r32)
            # a handful of output values (1x1 images, one-cell detectors): rel-L2 of one fp32 sum
            # with cancellation is not a projector property; allow 10x there
            ok = e <= (tol if a32[0].size >= 16 else 10 * tol)
        desc = (f"{name} {kind} s={s} na={g.n_angles} nd={g.det_count} sp={g.det_spacing:.3f} B={B} step={step}"
                f"{' host' if host_path else ''}")
        if e > worst[dt][0]:
            worst[dt] = (e, desc)
        if not ok:
            fails += 1
            print(f"FAIL case {c}: {desc} {dt} rel_l2={e:.3e}", flush=True)
print(f"stress parity: {ran} of {n_cases} cases run, {fails} failures, worst rel-L2 fp32 {worst['fp32'][0]:.2e} "
      f"({worst['fp32'][1]}), fp16 {worst['fp16'][0]:.2e} ({worst['fp16'][1]}), fp64 {worst['fp64'][0]:.2e}, "
      f"{time.time() - t0:.0f} s")
sys.exit(1 if fails else 0)
