"""Per-image device time of the cfg2 projector pair against the batch size
(small batches: grid fill / tail effects).  python tools/batch_probe.py [workload]"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2009_14788_b200 as rk  # noqa: E402
from paper_2009_14788_b200 import _lib  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "par512"
k, s, na, stop, nd, src, _ = bench.WORKLOADS[wl]
ang = rk.angles_linspace(0.0, stop, na)
g = rk.make_parallel(s, ang, nd) if k == "parallel" else rk.make_fanbeam(s, ang, src, det_count=nd)
plan = rk.get_plan(g, None, 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
V = ctypes.c_void_p
out = {}
for b in (1, 2, 4, 8, 12, 16, 24, 32, 64, 128):
    x = torch.rand(b, s, s, device="cuda")
    sino = torch.empty(b, na, nd, device="cuda")
    img = torch.empty(b, s, s, device="cuda")
    fns = {"forward": lambda: _lib.check(_lib.lib.rk_forward(plan.handle, _lib.RK_F32, V(x.data_ptr()), b,
                                                             V(sino.data_ptr()), V(st.cuda_stream))),
           "backproject": lambda: _lib.check(_lib.lib.rk_backproject(plan.handle, _lib.RK_F32, V(sino.data_ptr()), b,
                                                                     V(img.data_ptr()), V(st.cuda_stream)))}
    res = {}
    for name, fn in fns.items():
        for _ in range(3):
            fn()
        ts = []
        for i in range(9):
            flush.fill_(i)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        res[name + "_ms"] = ts[4]
        res[name + "_us_per_image"] = 1e3 * ts[4] / b
    out[b] = res
print(json.dumps({"workload": wl, "by_batch": out}, indent=1))
