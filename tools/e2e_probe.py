"""Host-buffer (e2e) path breakdown at cfg2: forward_host and backproject_host
wall times vs their device kernels, and raw pinned copy bandwidth."""
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

B, s, na, nd = 128, 512, 512, 512
g = rk.make_parallel(s, rk.angles_linspace(0, math.pi, na))
plan = rk.get_plan(g, None, 0)
h_img = torch.rand(B, s, s).pin_memory()
h_sino = torch.empty(B, na, nd).pin_memory()
h_out = torch.empty(B, s, s).pin_memory()
V = ctypes.c_void_p


def fwd():
    _lib.check(_lib.lib.rk_forward_host(plan.handle, _lib.RK_F32, V(h_img.data_ptr()), B, V(h_sino.data_ptr())))


def bp():
    _lib.check(_lib.lib.rk_backproject_host(plan.handle, _lib.RK_F32, V(h_sino.data_ptr()), B, V(h_out.data_ptr())))


def wall(fn, reps=5):
    fn()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) / reps * 1e3


res = {"forward_host_ms": wall(fwd), "backproject_host_ms": wall(bp)}
d = torch.empty(B, s, s, device="cuda")
d.copy_(h_img)
h_out.copy_(d)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    d.copy_(h_img, non_blocking=True)
torch.cuda.synchronize()
res["h2d_GBps"] = 5 * h_img.numel() * 4 / (time.perf_counter() - t) / 1e9
t = time.perf_counter()
for _ in range(5):
    h_out.copy_(d, non_blocking=True)
torch.cuda.synchronize()
res["d2h_GBps"] = 5 * h_img.numel() * 4 / (time.perf_counter() - t) / 1e9
print(json.dumps(res))
