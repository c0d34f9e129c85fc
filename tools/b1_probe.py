"""Batch-1 timings (single-lane kernels vs packed): forward / backprojection
at 512^2 (parallel, fan) and the paper's ADMM on one image.
Usage: python tools/b1_probe.py   (RK_SINGLE_LANE=0 forces the packed kernels)"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402
from paper_2009_14788_b200.phantom import shepp_logan  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


res = {"single_lane": os.environ.get("RK_SINGLE_LANE", "1") != "0"}
x = torch.from_numpy(shepp_logan(512)[None]).cuda()
for name, g in (("par512", rk.make_parallel(512, rk.angles_linspace(0, math.pi, 512))),
                ("fan512", rk.make_fanbeam(512, rk.angles_linspace(0, 2 * math.pi, 512), 512.0))):
    y = rk.forward(g, x)
    res[name] = {"forward_ms": timed(lambda: rk.forward(g, x)), "backprojection_ms": timed(lambda: rk.backprojection(g, y))}
ga = rk.make_parallel(512, [(i * 100.0 / 512 - 50.0) * math.pi / 180.0 for i in range(512)])
plan = rk.make_plan(512, 512, [0.5] * 5)
ya = rk.forward(ga, x)
op = rk.projector_operator(ga)
rk.admm_reconstruct(op, plan, ya, rk.AdmmParams(outer_iterations=1))
res["admm_b1_s"] = timed(lambda: rk.admm_reconstruct(op, plan, ya, rk.AdmmParams(outer_iterations=50,
                                                                                 inner_cg_iterations=50)), reps=1) / 1e3
print(json.dumps(res))
