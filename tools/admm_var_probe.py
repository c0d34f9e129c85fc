import math, time, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2009_14788_b200 as rk
from paper_2009_14788_b200.phantom import shepp_logan
ga = rk.make_parallel(512, [(i * 100.0 / 512 - 50.0) * math.pi / 180.0 for i in range(512)])
op = rk.projector_operator(ga)
plan = rk.make_plan(512, 512, [0.5] * 5)
x = torch.from_numpy(shepp_logan(512)[None]).cuda()
y = rk.forward(ga, x)
for run in range(6):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter(); a.record()
    rk.admm_reconstruct(op, plan, y, rk.AdmmParams(outer_iterations=50 if run else 20, inner_cg_iterations=50))
    b.record(); torch.cuda.synchronize()
    print(run, "wall %.1f ms  events %.1f ms" % ((time.perf_counter() - t) * 1e3, a.elapsed_time(b)), flush=True)

# per outer iteration (rk_admm_iterate(1) each, device events around it)
import ctypes
from paper_2009_14788_b200 import _lib, _arrays as A
rplan = rk.get_plan(ga, None, 0)
sh = plan._device_handle(0)
h = ctypes.c_void_p()
stream = A.stream_of(y)
_lib.check(_lib.lib.rk_admm_create(rplan.handle, sh, _lib.RK_F32, A.ptr(y), 1, 0.02, 0.1, None, 50, stream, ctypes.byref(h)))
times = []
for it in range(150):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    failed = ctypes.c_int64(-1)
    _lib.check(_lib.lib.rk_admm_iterate(h, 1, ctypes.byref(failed), stream), failed.value)
    b.record(); torch.cuda.synchronize()
    times.append(a.elapsed_time(b))
_lib.lib.rk_admm_destroy(h)
t = np.array(times)
print("per-iteration ms: median %.2f min %.2f max %.2f; > 1.5x median at" % (np.median(t), t.min(), t.max()),
      [int(i) for i in np.where(t > 1.5 * np.median(t))[0]], [round(float(v), 1) for v in t[t > 1.5 * np.median(t)]])
