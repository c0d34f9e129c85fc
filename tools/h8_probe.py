"""fp16-storage timings: forward / backprojection at 512^2 (parallel, fan; batch 128)
and FBP at config 4, for the half8 layout vs the float4 one (RK_H8=0)."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


res = {"h8": os.environ.get("RK_H8", "1") != "0"}
x = torch.rand(128, 512, 512, device="cuda").half()
for name, g in (("par512", rk.make_parallel(512, rk.angles_linspace(0, math.pi, 512))),
                ("fan512", rk.make_fanbeam(512, rk.angles_linspace(0, 2 * math.pi, 512), 512.0))):
    y = rk.forward(g, x)
    res[name] = {"forward_ms": timed(lambda: rk.forward(g, x)), "backprojection_ms": timed(lambda: rk.backprojection(g, y))}
del x
for nd in (1024, 1449):
    g = rk.make_parallel(1024, rk.angles_linspace(0.0, math.pi, 720), nd)
    s = torch.rand(64, 720, nd, device="cuda").half()
    res[f"fbp1024_nd{nd}_ms"] = timed(lambda: rk.fbp(g, s))
print(json.dumps(res))
