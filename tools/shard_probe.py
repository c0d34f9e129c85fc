"""Strong-scaling preview on one GPU: the cfg2 step at the per-GPU batch of
N = 1, 2, 4, 8 ranks (128 / N images), device-timed per kernel, so the
per-rank efficiency of the multi-GPU bench can be read off one B200.

  python tools/shard_probe.py [workload]
"""
import ctypes
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2009_14788_b200 as rk  # noqa: E402
from paper_2009_14788_b200 import _lib  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "par512"
k, s, na, stop, nd, src, B = bench.WORKLOADS[wl]
ang = rk.angles_linspace(0.0, stop, na)
g = rk.make_parallel(s, ang, nd) if k == "parallel" else rk.make_fanbeam(s, ang, src, det_count=nd)
plan = rk.get_plan(g, None, 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
V = ctypes.c_void_p
out = {}
for n in (1, 2, 4, 8):
    b = math.ceil(B / n)
    x = torch.rand(b, s, s, device="cuda")
    sino = torch.empty(b, na, nd, device="cuda")
    img = torch.empty(b, s, s, device="cuda")

    def fwd():
        _lib.check(_lib.lib.rk_forward(plan.handle, _lib.RK_F32, V(x.data_ptr()), b, V(sino.data_ptr()),
                                       V(st.cuda_stream)))

    def bp():
        _lib.check(_lib.lib.rk_backproject(plan.handle, _lib.RK_F32, V(sino.data_ptr()), b, V(img.data_ptr()),
                                           V(st.cuda_stream)))

    res = {}
    for name, fn in (("forward", fwd), ("backproject", bp), ("step", lambda: (fwd(), bp()))):
        for _ in range(3):
            fn()
        tot = []
        for i in range(10):
            flush.fill_(i)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            tot.append(e0.elapsed_time(e1))
        tot.sort()
        res[name + "_ms"] = tot[len(tot) // 2]
    res["per_gpu_batch"] = b
    res["aggregate_images_per_s"] = n * b / (res["step_ms"] * 1e-3)
    out[f"N{n}"] = res
base = out["N1"]["aggregate_images_per_s"]
for n in (1, 2, 4, 8):
    out[f"N{n}"]["efficiency_vs_N1"] = out[f"N{n}"]["aggregate_images_per_s"] / (n * base)
print(json.dumps({"workload": wl, **out}, indent=1))
