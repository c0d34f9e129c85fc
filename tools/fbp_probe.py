"""Per-kernel-kind device time of FBP at config 4 (1024^2, 720 angles, batch 64):
filter vs backprojection vs packing.  Usage: python tools/fbp_probe.py"""
import ctypes
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402
from paper_2009_14788_b200 import _lib  # noqa: E402


def kstats():
    st = _lib.RkKernelStats()
    _lib.check(_lib.lib.rk_profiling_read(ctypes.byref(st), 1))
    return {k: round(float(st.ms[i]) / max(1, int(st.timed[i])), 4) for i, k in enumerate(_lib.KERNEL_KINDS)
            if st.launches[i]}


res = {}
for nd in (1024, 1449):
    g = rk.make_parallel(1024, rk.angles_linspace(0.0, math.pi, 720), nd)
    sino = torch.rand(64, 720, nd, device="cuda")
    for dt in (torch.float32, torch.float16):
        s_ = sino.to(dt)
        rk.fbp(g, s_)
        torch.cuda.synchronize()
        _lib.check(_lib.lib.rk_profiling_enable(1))
        kstats()
        for _ in range(3):
            rk.fbp(g, s_)
        torch.cuda.synchronize()
        _lib.check(_lib.lib.rk_profiling_enable(0))
        res[f"nd{nd}_{str(dt).split('.')[-1]}"] = kstats()
print(json.dumps(res))
