"""Minimal driver for ncu: shearlet analysis + synthesis at 512^2, 5 scales, batch 8."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
plan = rk.make_plan(512, 512, [0.5] * 5)
x = torch.rand(B, 512, 512, device="cuda")
for _ in range(2):
    c = rk.forward(plan, x)
    rk.backward(plan, c)
torch.cuda.synchronize()
print("done")
