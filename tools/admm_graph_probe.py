"""Per-outer-iteration device time of ADMM (paper config) through rk_admm_iterate: direct launches
vs graph replays (RK_ADMM_GRAPH), after the first (eager + capture) call.  python tools/admm_graph_probe.py"""
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
from paper_2009_14788_b200 import _arrays as A, _lib  # noqa: E402
from paper_2009_14788_b200.phantom import shepp_logan  # noqa: E402
from paper_2009_14788_b200.projector import get_plan  # noqa: E402

ga = rk.make_parallel(512, [(i * 100.0 / 512 - 50.0) * math.pi / 180.0 for i in range(512)])
op = rk.projector_operator(ga)
plan = rk.make_plan(512, 512, [0.5] * 5)
x = torch.from_numpy(np.stack([shepp_logan(512) * ((e + 1) / 8.0) for e in range(8)])).cuda()
res = {}
for b in (1, 8):
    y = rk.forward(ga, x[:b]).contiguous()
    rplan = get_plan(ga, None, 0)
    sh = plan._device_handle(0)
    for mode in ("1", "0", "1", "0"):
        os.environ["RK_ADMM_GRAPH"] = mode
        h = ctypes.c_void_p()
        st = A.stream_of(y)
        _lib.check(_lib.lib.rk_admm_create(rplan.handle, sh, _lib.RK_F32, A.ptr(y), b, 0.02, 0.1, None, 50, st,
                                           ctypes.byref(h)))
        failed = ctypes.c_int64(-1)
        t0 = time.perf_counter()
        _lib.check(_lib.lib.rk_admm_iterate(h, 1, ctypes.byref(failed), st))
        t1 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(_lib.lib.rk_admm_iterate(h, 20, ctypes.byref(failed), st))
        e1.record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        _lib.lib.rk_admm_destroy(h)
        res.setdefault(f"b{b}_graph{mode}", []).append(
            {"first_call_ms": round(1e3 * (t1 - t0), 1), "per_iter_ms_device": round(e0.elapsed_time(e1) / 20, 3),
             "per_iter_ms_wall": round(1e3 * (t2 - t1) / 20, 3)})
print(json.dumps(res, indent=1))
