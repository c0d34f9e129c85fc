"""One-shot latency breakdown at config 2 (parallel 512^2 / 512 angles): plan creation,
forward-schedule preparation (planned: cold cache; read: warm cache) and the first
rk_forward_host of one image.  python tools/first_call_probe.py [reps]"""
import ctypes
import json
import math
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402
from paper_2009_14788_b200 import _lib  # noqa: E402
from paper_2009_14788_b200.projector import Plan  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
x = np.random.rand(1, 512, 512).astype(np.float32)
y = np.empty((1, 512, 512), np.float32)
res = []
for name, g in (("par512", rk.make_parallel(512, rk.angles_linspace(0.0, math.pi, 512), 512)),
                ("fan512", rk.make_fanbeam(512, rk.angles_linspace(0.0, 2 * math.pi, 512), 512.0))):
    for r in range(reps):
        os.environ["RK_PLAN_CACHE"] = tempfile.mkdtemp()
        for key in ("cold", "warm"):
            t0 = time.perf_counter()
            p = Plan(g, 1.0, 0)
            t1 = time.perf_counter()
            p.prepare()
            t2 = time.perf_counter()
            _lib.check(_lib.lib.rk_forward_host(p.handle, _lib.RK_F32, ctypes.c_void_p(x.ctypes.data), 1,
                                                ctypes.c_void_p(y.ctypes.data)))
            t3 = time.perf_counter()
            _lib.check(_lib.lib.rk_forward_host(p.handle, _lib.RK_F32, ctypes.c_void_p(x.ctypes.data), 1,
                                                ctypes.c_void_p(y.ctypes.data)))
            t4 = time.perf_counter()
            res.append({"geom": name, "rep": r, "cache": key, "from_cache": p.info()["schedule_from_cache"],
                        "create_ms": 1e3 * (t1 - t0), "prepare_ms": 1e3 * (t2 - t1),
                        "first_forward_ms": 1e3 * (t3 - t2), "second_forward_ms": 1e3 * (t4 - t3),
                        "total_ms": 1e3 * (t3 - t0)})
            del p
for r in res:
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}))
