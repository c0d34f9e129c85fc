"""GPU probe for the shearlet transform and ADMM: parity numbers against the
reference oracle (small sizes) and device timings at 512^2 with per-kernel-kind
breakdowns.  Usage: python tools/probe_admm.py [--no-parity] [--out FILE]"""
import argparse
import ctypes
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402
from paper_2009_14788_b200 import _lib  # noqa: E402


def limited(n):
    return [(i * 100.0 / n - 50.0) * math.pi / 180.0 for i in range(n)]


def kstats(reset=True):
    st = _lib.RkKernelStats()
    _lib.check(_lib.lib.rk_profiling_read(ctypes.byref(st), int(reset)))
    return {k: {"launches": int(st.launches[i]), "ms": float(st.ms[i])} for i, k in enumerate(_lib.KERNEL_KINDS)
            if st.launches[i]}


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(reps):
        fn()
    ev1.record()
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    res = {}
    if not a.no_parity:
        from oracle import Geom, RefOracle, rel_l2

        ref = RefOracle()
        for s, na, alphas, outer, inner, batch in [(32, 32, [0.5] * 3, 6, 20, 1), (64, 48, [0.5] * 2, 4, 15, 3),
                                                   (64, 64, [0.5] * 3, 20, 50, 1)]:
            ang = limited(na)
            g = rk.make_parallel(s, ang)
            x = np.concatenate([ref.shepp_logan(s, np.float64) * (1 - 0.25 * e) for e in range(batch)])
            y = rk.forward(g, torch.from_numpy(x.astype(np.float32)).cuda()).cpu().numpy()
            rec = rk.admm_reconstruct(rk.projector_operator(g), rk.make_plan(s, s, alphas), torch.from_numpy(y).cuda(),
                                      rk.AdmmParams(outer_iterations=outer, inner_cg_iterations=inner)).cpu().numpy()
            rr = ref.admm(Geom("parallel", s, np.asarray(ang)), y, alphas, 0.02, 0.1, outer, inner)
            res[f"admm_rel_{s}_{outer}x{inner}_b{batch}"] = rel_l2(rec, rr)
        for n, alphas in [(64, [0.5] * 5), (128, [0.5] * 4)]:
            x = np.random.default_rng(0).standard_normal((2, n, n)).astype(np.float32)
            p = rk.make_plan(n, n, alphas)
            c = rk.forward(p, torch.from_numpy(x).cuda()).cpu().numpy()
            cr = ref.shearlet_forward(x, alphas)
            res[f"shearlet_fwd_rel_{n}"] = rel_l2(c, cr)
            b = rk.backward(p, torch.from_numpy(cr).cuda()).cpu().numpy()
            res[f"shearlet_bwd_rel_{n}"] = rel_l2(b, ref.shearlet_backward(cr, alphas))
    print(json.dumps(res), flush=True)

    # ---- timings at 512^2, 5 scales (59 coefficients)
    _lib.check(_lib.lib.rk_profiling_enable(1))
    n = 512
    plan = rk.make_plan(n, n, [0.5] * 5)
    for B in (1, 8):
        x = torch.rand(B, n, n, device="cuda")
        c = rk.forward(plan, x)
        kstats()
        tf = timed(lambda: rk.forward(plan, x))
        kf = kstats()
        tb = timed(lambda: rk.backward(plan, c))
        kb = kstats()
        coeff_bytes = B * plan.n_coeff * n * n * 4
        res[f"shearlet512_b{B}"] = {"fwd_ms": tf, "bwd_ms": tb, "coeff_GBps_fwd": coeff_bytes / tf / 1e6,
                                   "coeff_GBps_bwd": coeff_bytes / tb / 1e6, "k_fwd": kf, "k_bwd": kb}
        print(json.dumps({f"shearlet512_b{B}": res[f"shearlet512_b{B}"]}), flush=True)
        del c
    for na in (512,):
        ang = limited(na)
        g = rk.make_parallel(n, ang)
        op = rk.projector_operator(g)
        for B in (1, 8, 32):
            x = torch.rand(B, n, n, device="cuda")
            y = rk.forward(g, x)
            prm = rk.AdmmParams(outer_iterations=2, inner_cg_iterations=50)
            rk.admm_reconstruct(op, plan, y, prm)
            torch.cuda.synchronize()
            kstats()
            t0 = time.perf_counter()
            ms = timed(lambda: rk.admm_reconstruct(op, plan, y, prm), reps=1)
            wall = time.perf_counter() - t0
            k = kstats()
            per_outer = ms / 2
            res[f"admm512_na{na}_b{B}"] = {"ms_2outer": ms, "ms_per_outer": per_outer,
                                          "s_per_image_50x50": per_outer * 50 / 1000 / B, "kernels": k}
            print(json.dumps({f"admm512_na{na}_b{B}": res[f"admm512_na{na}_b{B}"]}), flush=True)
            del x, y
            torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
