"""Run-to-run spread of the paper's ADMM on one image (512^2, 50 x 50): five back-to-back
reconstructions in one process (the first ones run while the GPU clocks ramp).
Usage: python tools/admm_var.py"""
import math, sys, time, os
sys.path.insert(0, os.getcwd())
import torch, paper_2009_14788_b200 as rk
from paper_2009_14788_b200.phantom import shepp_logan
x = torch.from_numpy(shepp_logan(512)[None]).cuda()
ga = rk.make_parallel(512, [(i * 100.0 / 512 - 50.0) * math.pi / 180.0 for i in range(512)])
plan = rk.make_plan(512, 512, [0.5] * 5)
ya = rk.forward(ga, x); op = rk.projector_operator(ga)
rk.admm_reconstruct(op, plan, ya, rk.AdmmParams(outer_iterations=1))
for i in range(5):
    torch.cuda.synchronize(); t = time.perf_counter()
    rk.admm_reconstruct(op, plan, ya, rk.AdmmParams(outer_iterations=50, inner_cg_iterations=50))
    torch.cuda.synchronize(); print("admm b1 s", round(time.perf_counter() - t, 3), flush=True)
