"""Wall time of each phase of one ADMM call (create / iterate(50) / read / destroy), repeated:
where the run-to-run variance of admm_reconstruct comes from.  python tools/admm_phase_probe.py [batch]"""
import ctypes
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402
from paper_2009_14788_b200 import _arrays as A  # noqa: E402
from paper_2009_14788_b200 import _lib  # noqa: E402
from paper_2009_14788_b200.phantom import shepp_logan  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ga = rk.make_parallel(512, [(i * 100.0 / 512 - 50.0) * math.pi / 180.0 for i in range(512)])
plan = rk.make_plan(512, 512, [0.5] * 5)
y = rk.forward(ga, torch.from_numpy(np.stack([shepp_logan(512)] * B)).cuda()).contiguous()
rplan = rk.get_plan(ga, None, 0)
sh = plan._device_handle(0)
stream = A.stream_of(y)
out = torch.empty(B, 512, 512, device="cuda")
for run in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = ctypes.c_void_p()
    _lib.check(_lib.lib.rk_admm_create(rplan.handle, sh, _lib.RK_F32, A.ptr(y), B, 0.02, 0.1, None, 50, stream,
                                       ctypes.byref(h)))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    failed = ctypes.c_int64(-1)
    _lib.check(_lib.lib.rk_admm_iterate(h, 50, ctypes.byref(failed), stream), failed.value)
    t2 = time.perf_counter()
    _lib.check(_lib.lib.rk_admm_read(h, 0, _lib.RK_F32, A.ptr(out), stream))
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    _lib.lib.rk_admm_destroy(h)
    t4 = time.perf_counter()
    print(f"B={B} run {run}: create {1e3 * (t1 - t0):.1f} ms, iterate(50) {1e3 * (t2 - t1):.1f} ms, "
          f"read {1e3 * (t3 - t2):.1f} ms, destroy {1e3 * (t4 - t3):.1f} ms", flush=True)
