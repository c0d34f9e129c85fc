"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once at tiny sizes — packed and single-lane projectors
(parallel, fan fp32 map, fan fp64 map), filter / FBP, fused solvers, shearlet
analysis / synthesis and one ADMM iteration.  Usage: python tools/sanitize_probe.py"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402

dev = torch.device("cuda", 0)
s, na = 32, 20
geoms = [rk.make_parallel(s, rk.angles_linspace(0.0, math.pi, na)),
         rk.make_fanbeam(s, rk.angles_linspace(0.0, 2 * math.pi, na), 2.0 * s),
         rk.make_fanbeam(s, rk.angles_linspace(0.0, 2 * math.pi, na), 24.0, det_distance=80.0)]
for g in geoms:
    for B in (1, 5):
        x = torch.rand(B, s, s, device=dev)
        y = rk.forward(g, x)
        rk.backprojection(g, y)
        rk.forward(g, x.half())
g = geoms[0]
y = rk.forward(g, torch.rand(3, s, s, device=dev))
rk.fbp(g, y)
op = rk.projector_operator(g)
rk.landweber(op, y, torch.zeros(3, s, s, device=dev), 1e-3, 2)
rk.cgne(op, torch.zeros(3, s, s, device=dev), y, 2)
plan = rk.make_plan(s, s, [0.5, 0.5])
c = rk.forward(plan, torch.rand(2, s, s, device=dev))
rk.backward(plan, c)
rk.admm_reconstruct(op, plan, y[:1], rk.AdmmParams(outer_iterations=1, inner_cg_iterations=2))
torch.cuda.synchronize()
print("sanitize probe done")
