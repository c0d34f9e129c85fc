import ctypes, json, math, os, sys, tempfile, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2009_14788_b200 as rk
from paper_2009_14788_b200 import _lib
from paper_2009_14788_b200.projector import Plan
g = rk.make_parallel(512, rk.angles_linspace(0.0, math.pi, 512), 512)
x = np.random.rand(1, 512, 512).astype(np.float32); y = np.empty((1, 512, 512), np.float32)
xd = torch.from_numpy(x).cuda(); yd = torch.empty(1, 512, 512, device='cuda')
os.environ["RK_PLAN_CACHE"] = tempfile.mkdtemp()
Plan(g, 1.0, 0).prepare()
def ms(f):
    torch.cuda.synchronize(); t = time.perf_counter(); f(); torch.cuda.synchronize(); return round(1e3 * (time.perf_counter() - t), 2)
for r in range(4):
    out = {}
    p = None
    def mk():
        global p; p = Plan(g, 1.0, 0)
    out['create'] = ms(mk)
    out['prepare'] = ms(lambda: p.prepare())
    out['dev_fwd1'] = ms(lambda: _lib.check(_lib.lib.rk_forward(p.handle, 1, ctypes.c_void_p(xd.data_ptr()), 1, ctypes.c_void_p(yd.data_ptr()), None)))
    out['dev_fwd2'] = ms(lambda: _lib.check(_lib.lib.rk_forward(p.handle, 1, ctypes.c_void_p(xd.data_ptr()), 1, ctypes.c_void_p(yd.data_ptr()), None)))
    out['host_fwd1'] = ms(lambda: _lib.check(_lib.lib.rk_forward_host(p.handle, 1, ctypes.c_void_p(x.ctypes.data), 1, ctypes.c_void_p(y.ctypes.data))))
    out['host_fwd2'] = ms(lambda: _lib.check(_lib.lib.rk_forward_host(p.handle, 1, ctypes.c_void_p(x.ctypes.data), 1, ctypes.c_void_p(y.ctypes.data))))
    out['destroy'] = ms(lambda: globals().pop('p'))
    print(json.dumps(out), flush=True)
