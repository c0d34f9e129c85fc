"""ADMM (paper config: 512^2, 100 degree arc, 512 angles, 5 scales, 50 x 50) seconds per image,
outer iterations replayed as a CUDA graph (RK_ADMM_GRAPH=1) vs direct launches (=0), 3 runs each.
python tools/admm_graph_ab.py"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402
from paper_2009_14788_b200.phantom import shepp_logan  # noqa: E402

ga = rk.make_parallel(512, [(i * 100.0 / 512 - 50.0) * math.pi / 180.0 for i in range(512)])
op = rk.projector_operator(ga)
plan = rk.make_plan(512, 512, [0.5] * 5)
x = torch.from_numpy(np.stack([shepp_logan(512) * ((e + 1) / 8.0) for e in range(8)])).cuda()
out = {}
for b in (1, 8):
    y = rk.forward(ga, x[:b])
    for mode in ("1", "0", "1", "0"):
        os.environ["RK_ADMM_GRAPH"] = mode
        rk.admm_reconstruct(op, plan, y, rk.AdmmParams(outer_iterations=10, inner_cg_iterations=50))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = rk.admm_reconstruct(op, plan, y, rk.AdmmParams(outer_iterations=50, inner_cg_iterations=50))
        e1.record()
        torch.cuda.synchronize()
        out.setdefault(f"b{b}_graph{mode}", []).append(round(e0.elapsed_time(e1) * 1e-3 / b, 4))
print(json.dumps(out))
