"""Ramp filter / FBP at large detector counts (the two-CTA cluster kernel, P = 2^14, 2^15)
against the reference: python tools/big_filter_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402
from oracle import Geom, default_oracle, rel_l2  # noqa: E402

orc = default_oracle()
fails = 0
for nd in (3, 4096, 4097, 6000, 8192, 9000, 16384, 16385):
    for dt, tol in ((np.float32, 1e-5), (np.float16, 1e-3), (np.float64, 1e-5)):
        y = (np.random.default_rng(nd).standard_normal((5, 3, nd)) * (0.01 if dt == np.float16 else 1)).astype(dt)
        try:
            for kind in ("ram-lak", "hann"):
                f = rk.filter_sinogram(torch.from_numpy(y).cuda(), rk.make_filter(rk.filter_kind_from_name(kind), nd))
                e = rel_l2(f.cpu().numpy().astype(np.float64), orc.filter_sinogram(y, kind).astype(np.float64))
                ok = e <= tol
                fails += not ok
                print(nd, np.dtype(dt).name, kind, "filter rel-L2 %.2e" % e, "ok" if ok else "FAIL", flush=True)
        except rk.ValidationError as ex:
            print(nd, "ValidationError", ex)
# FBP through the packed (float4 / half8) epilogues
for nd, dt, tol in ((6000, np.float32, 1e-5), (9000, np.float32, 1e-5), (6000, np.float16, 1e-3)):
    s = 64
    g = rk.make_parallel(s, rk.angles_linspace(0.0, np.pi, 8), nd, 0.02)
    y = (np.random.default_rng(1).standard_normal((9, 8, nd)) * (0.01 if dt == np.float16 else 1)).astype(dt)
    fb = rk.fbp(g, torch.from_numpy(y).cuda()).cpu().numpy()
    e = rel_l2(fb.astype(np.float64), orc.fbp(Geom("parallel", s, np.asarray(g.angles), nd, 0.02), y).astype(np.float64))
    fails += not (e <= tol)
    print("fbp", nd, np.dtype(dt).name, "rel-L2 %.2e" % e, "ok" if e <= tol else "FAIL", flush=True)
print("big filter probe:", fails, "failures")
sys.exit(1 if fails else 0)
