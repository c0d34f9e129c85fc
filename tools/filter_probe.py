import ctypes, json, math, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2009_14788_b200 as rk
from paper_2009_14788_b200 import _lib
def kstats():
    st = _lib.RkKernelStats(); _lib.check(_lib.lib.rk_profiling_read(ctypes.byref(st), 1))
    return {k: round(float(st.ms[i]) / max(1, int(st.timed[i])), 4) for i, k in enumerate(_lib.KERNEL_KINDS) if st.launches[i]}
res = {}
for nd in (1024, 1449):
    g = rk.make_parallel(1024, rk.angles_linspace(0.0, math.pi, 720), nd)
    f = rk.make_filter("ram-lak", nd)
    sino = torch.rand(64, 720, nd, device="cuda")
    for dt in (torch.float32, torch.float16):
        s_ = sino.to(dt)
        for name, fn in (("fbp", lambda: rk.fbp(g, s_)), ("filt", lambda: rk.filter_sinogram(s_, f))):
            fn(); torch.cuda.synchronize()
            _lib.check(_lib.lib.rk_profiling_enable(1)); kstats()
            for _ in range(3): fn()
            torch.cuda.synchronize(); _lib.check(_lib.lib.rk_profiling_enable(0))
            res[f"{name}_nd{nd}_{str(dt).split('.')[-1]}"] = kstats().get("filter")
print(json.dumps(res))
