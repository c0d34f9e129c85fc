"""Randomised parity sweep of the §8(f) widening (GPU vs the reference compiled in place):
estimate_alpha, fused Landweber and CGNE on random small geometries / batches / storage
dtypes, the shearlet transform on random power-of-two grids and scale lists, and a short
ADMM.  Prints one line per failure and a summary; exit 1 on any failure.

  python tools/stress_solvers.py [n_cases] [seed]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402
from oracle import Geom, default_oracle, rel_l2  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
orc = default_oracle()
rs = np.random.default_rng(seed)
fails, t0, worst = 0, time.time(), {}


def check(name, a, r, tol, desc):
    global fails
    a64, r64 = np.asarray(a, np.float64), np.asarray(r, np.float64)
    e = rel_l2(a64, r64) if np.abs(r64).max() > 0 else float(np.abs(a64).max())
    if e >= worst.get(name, (0.0, ""))[0]:
        worst[name] = (e, desc)
    if not e <= tol:
        fails += 1
        print(f"FAIL {name}: {desc} rel_l2={e:.3e} (tol {tol:g})", flush=True)


for c in range(n_cases):
    s = int(rs.choice([16, 24, 32, 48, 64, 80]))
    kind = "fan" if rs.random() < 0.4 else "par"
    na = int(rs.integers(8, 64))
    ang = list(np.linspace(0.0, 2 * np.pi if kind == "fan" else np.pi, na, endpoint=False)) if rs.random() < 0.6 \
        else list(rs.uniform(-4, 4, na))
    g = rk.make_parallel(s, ang) if kind == "par" else rk.make_fanbeam(s, ang, float(s) * float(rs.uniform(1.5, 3.0)))
    og = (Geom("fanbeam", s, np.asarray(g.angles), g.det_count, g.det_spacing, g.source_distance, g.det_distance)
          if kind == "fan" else Geom("parallel", s, np.asarray(g.angles), g.det_count, g.det_spacing))
    B = int(rs.choice([1, 2, 4, 5, 9]))
    dt = np.float32 if rs.random() < 0.8 else np.float64
    desc = f"{kind} s={s} na={na} B={B} {np.dtype(dt).name}"
    op = rk.projector_operator(g)
    # estimate_alpha (batch 1, fp64 power iteration of the fp32 operator)
    a_gpu, a_ref = rk.estimate_alpha(op, 20, 0), orc.estimate_alpha(og, 20, 0)
    check("estimate_alpha", a_gpu, a_ref, 1e-5, desc)
    x = (rs.uniform(0, 1, (B, s, s))).astype(dt)
    y = orc.forward(og, x)
    guess = np.zeros_like(x)
    it = int(rs.integers(1, 12))
    lw = rk.landweber(op, torch.from_numpy(y).cuda(), torch.from_numpy(guess).cuda(), 0.95 * a_ref, it).cpu().numpy()
    check("landweber", lw, orc.landweber(og, y, guess, 0.95 * a_ref, it), 1e-5, desc + f" it={it}")
    ci = int(rs.integers(1, 12))
    cg = rk.cgne(op, torch.from_numpy(guess).cuda(), torch.from_numpy(y).cuda(), ci).cpu().numpy()
    check("cgne", cg, orc.cgne(og, y, guess, ci), 1e-3, desc + f" it={ci}")

# shearlets on random power-of-two grids and scale lists
for c in range(max(4, n_cases // 4)):
    n = int(rs.choice([2, 3, 4, 8, 10, 16, 24, 32, 50, 64, 100, 128, 256]))  # any square grid
    alphas = list(np.round(rs.uniform(0, 1, int(rs.integers(1, 6))), 3))
    B = int(rs.integers(1, 4))
    dt = np.float32 if rs.random() < 0.7 else np.float64
    x = rs.standard_normal((B, n, n)).astype(dt)
    p = rk.make_plan(n, n, alphas)
    cf = rk.forward(p, torch.from_numpy(x).cuda()).cpu().numpy()
    cr = orc.shearlet_forward(x, alphas)
    tol = 1e-12 if dt == np.float64 else 1e-5
    desc = f"n={n} alphas={alphas} B={B} {np.dtype(dt).name}"
    check("shearlet_forward", cf, cr, tol, desc)
    bk = rk.backward(p, torch.from_numpy(cr).cuda()).cpu().numpy()
    check("shearlet_backward", bk, orc.shearlet_backward(cr, alphas), tol, desc)

# a few short ADMMs (512-angle sinograms are the paper's; small here)
for c in range(max(2, n_cases // 10)):
    s = int(rs.choice([24, 32, 40, 64]))
    na = int(rs.integers(16, 48))
    ang = list(np.linspace(-np.pi / 4, np.pi / 4, na))
    g = rk.make_parallel(s, ang)
    og = Geom("parallel", s, np.asarray(g.angles), g.det_count, g.det_spacing)
    ph = orc.shepp_logan(s)
    y = orc.forward(og, ph)
    alphas = [0.5] * int(rs.integers(1, 4))
    outer, inner = int(rs.integers(2, 6)), int(rs.integers(2, 6))
    p0, p1 = float(rs.uniform(0.5, 2.0)), float(rs.uniform(0.05, 0.5))
    plan = rk.make_plan(s, s, alphas)
    params = rk.AdmmParams(p0=p0, p1=p1, outer_iterations=outer, inner_cg_iterations=inner)
    f = rk.admm_reconstruct(rk.projector_operator(g), plan, torch.from_numpy(y).cuda(), params).cpu().numpy()
    fr = orc.admm(og, y, alphas, p0, p1, outer, inner)
    check("admm", f, fr, 2e-4, f"s={s} na={na} alphas={alphas} outer={outer} inner={inner} p0={p0:.2f} p1={p1:.2f}")

print(f"stress solvers: {fails} failures in {time.time() - t0:.0f} s; worst "
      + ", ".join(f"{k} {v[0]:.1e}" for k, v in worst.items()))
sys.exit(1 if fails else 0)
