"""ADMM (paper config: 512^2, 100 degree arc, 512 angles, 5 scales, 50 x 50) seconds per image at batch 1 / 4 / 8,
with the per-kernel-kind device time of one run.  python tools/admm_ab.py"""
import ctypes
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402
from paper_2009_14788_b200 import _lib  # noqa: E402
from paper_2009_14788_b200.phantom import shepp_logan  # noqa: E402

ga = rk.make_parallel(512, [(i * 100.0 / 512 - 50.0) * math.pi / 180.0 for i in range(512)])
op = rk.projector_operator(ga)
plan = rk.make_plan(512, 512, [0.5] * 5)
x = torch.from_numpy(np.stack([shepp_logan(512) * ((e + 1) / 8.0) for e in range(8)])).cuda()
out = {}
for b in (1, 4, 8):
    y = rk.forward(ga, x[:b])
    rk.admm_reconstruct(op, plan, y, rk.AdmmParams(outer_iterations=20, inner_cg_iterations=50))
    torch.cuda.synchronize()
    st = _lib.RkKernelStats()
    _lib.check(_lib.lib.rk_profiling_read(ctypes.byref(st), 1))
    _lib.check(_lib.lib.rk_profiling_enable(1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rk.admm_reconstruct(op, plan, y, rk.AdmmParams(outer_iterations=50, inner_cg_iterations=50))
    e1.record()
    torch.cuda.synchronize()
    _lib.check(_lib.lib.rk_profiling_enable(0))
    _lib.check(_lib.lib.rk_profiling_read(ctypes.byref(st), 1))
    kinds = {k: round(float(st.ms[i]), 1) for i, k in enumerate(_lib.KERNEL_KINDS) if st.launches[i]}
    out[b] = {"s_per_image": e0.elapsed_time(e1) * 1e-3 / b, "kernel_ms": kinds}
print(json.dumps(out, indent=1))
