"""Extreme-geometry sweep: large images, many angles, very fine or very coarse detectors,
sources close to the image.  Reports failures (parity or exceptions) against the reference.
  python tools/stress_extreme.py [n_cases] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402
from oracle import Geom, default_oracle, rel_l2  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
orc = default_oracle()
rs = np.random.default_rng(seed)
fails, t0 = 0, time.time()
for c in range(n_cases):
    s = int(rs.choice([256, 384, 512, 700, 1024]))
    kind = "fan" if rs.random() < 0.5 else "par"
    na = int(rs.choice([3, 100, 360, 720, 1000]))
    sp = float(rs.choice([0.01, 0.05, 0.2, 0.5, 3.0, 9.0, 40.0]))
    nd = int(min(4096, max(2, rs.integers(2, int(1.5 * s * np.sqrt(2) / sp) + 3))))
    ang = list(np.linspace(0, 2 * np.pi if kind == "fan" else np.pi, na, endpoint=False))
    try:
        if kind == "par":
            g = rk.make_parallel(s, ang, nd, sp)
            og = Geom("parallel", s, np.asarray(g.angles), nd, sp)
        else:
            src = float(s) * float(rs.choice([0.72, 0.8, 1.0, 2.0, 10.0]))
            g = rk.make_fanbeam(s, ang, src, float(s) * float(rs.choice([0.5, 1.0, 4.0])), nd, sp)
            og = Geom("fanbeam", s, np.asarray(g.angles), nd, sp, g.source_distance, g.det_distance)
    except rk.ValidationError:
        continue
    desc = f"{kind} s={s} na={na} nd={nd} sp={sp} src={getattr(g, 'source_distance', None)}"
    x = rs.uniform(0, 1, (1, s, s)).astype(np.float32)
    y = rs.standard_normal((1, na, nd)).astype(np.float32)
    t1 = time.time()
    try:
        f = rk.forward(g, torch.from_numpy(x).cuda()).cpu().numpy()
        b = rk.backprojection(g, torch.from_numpy(y).cuda()).cpu().numpy()
    except Exception as exc:  # noqa: BLE001
        fails += 1
        print(f"FAIL {desc}: {type(exc).__name__}: {exc}", flush=True)
        continue
    tg = time.time() - t1
    ef = rel_l2(f, orc.forward(og, x)) if np.abs(f).max() > 0 else 0.0
    eb = rel_l2(b, orc.backprojection(og, y))
    ok = ef <= 1e-5 and eb <= 1e-5
    fails += not ok
    print(f"{'ok  ' if ok else 'FAIL'} {desc}: fwd {ef:.2e} bp {eb:.2e} (gpu {tg:.2f} s)", flush=True)
print(f"stress extreme: {fails} failures, {time.time() - t0:.0f} s")
sys.exit(1 if fails else 0)
