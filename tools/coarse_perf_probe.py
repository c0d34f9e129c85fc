import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2009_14788_b200 as rk
for kind, s, nd, sp in [('fan', 512, 128, None), ('fan', 512, 64, None), ('par', 512, 64, 8.0), ('par', 512, 512, None), ('fan', 512, 512, None)]:
    ang = rk.angles_linspace(0, np.pi if kind == 'par' else 2 * np.pi, 512)
    g = rk.make_parallel(s, ang, nd, sp) if kind == 'par' else rk.make_fanbeam(s, ang, 512.0, det_count=nd)
    x = torch.rand(16, s, s, device='cuda')
    y = rk.forward(g, x); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); y = rk.forward(g, x); b.record(); torch.cuda.synchronize()
    tf = a.elapsed_time(b)
    a.record(); z = rk.backprojection(g, y); b.record(); torch.cuda.synchronize()
    print(kind, s, nd, g.det_spacing, "forward %.2f ms  bp %.2f ms (batch 16)" % (tf, a.elapsed_time(b)), flush=True)
