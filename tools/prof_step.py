"""Minimal driver for ncu: a few forward + backprojection steps of a bench workload
through the C ABI (no timing, no oracle).
Usage: python tools/prof_step.py [workload] [steps] [batch] [f32|f16]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2009_14788_b200 as rk  # noqa: E402
from paper_2009_14788_b200 import _lib  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "par512"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
k, s, na, stop, nd, src, B = bench.WORKLOADS[wl]
B = int(sys.argv[3]) if len(sys.argv) > 3 else B
ang = rk.angles_linspace(0.0, stop, na)
g = rk.make_parallel(s, ang, nd) if k == "parallel" else rk.make_fanbeam(s, ang, src, det_count=nd)
half = len(sys.argv) > 4 and sys.argv[4] == "f16"
dt, code = (torch.float16, 0) if half else (torch.float32, 1)  # RK_F16 = 0, RK_F32 = 1
x = torch.rand(B, s, s, device="cuda").to(dt)
sino = torch.empty(B, na, nd, device="cuda", dtype=dt)
out = torch.empty(B, s, s, device="cuda", dtype=dt)
plan = rk.get_plan(g, None, 0)
for _ in range(steps):
    _lib.check(_lib.lib.rk_forward(plan.handle, code, ctypes.c_void_p(x.data_ptr()), B, ctypes.c_void_p(sino.data_ptr()), None))
    _lib.check(_lib.lib.rk_backproject(plan.handle, code, ctypes.c_void_p(sino.data_ptr()), B, ctypes.c_void_p(out.data_ptr()), None))
torch.cuda.synchronize()
print("done", wl, B, steps)
