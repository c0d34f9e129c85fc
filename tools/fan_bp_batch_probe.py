import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2009_14788_b200 as rk
g = rk.make_fanbeam(512, rk.angles_linspace(0, 2 * np.pi, 512), 512.0)
for B in (16, 128, 16, 4, 1, 8, 32):
    y = torch.rand(B, 512, 512, device='cuda')
    z = rk.backprojection(g, y); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); z = rk.backprojection(g, y); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print("fan bp batch", B, ["%.2f" % t for t in ts], "ms", flush=True)
