"""Minimal driver for ncu: FBP at config 4 (1024^2, 720 angles, nd 1024 or 1449, batch 64) through
the C ABI (rk_fbp: filter_kernel writes the packed sinogram, then the backprojection).
Usage: python tools/prof_fbp.py [nd] [steps] [f32|f16]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402

nd = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dt = torch.float16 if len(sys.argv) > 3 and sys.argv[3] == "f16" else torch.float32
g = rk.make_parallel(1024, rk.angles_linspace(0.0, math.pi, 720), nd)
sino = torch.rand(64, 720, nd, device="cuda").to(dt)
for _ in range(steps):
    rk.fbp(g, sino)
torch.cuda.synchronize()
print("done fbp", nd, steps)
