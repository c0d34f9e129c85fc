"""fp32 vs fp64 fan-beam backprojection map against the reference, by magnification
span / (spacing (D_so - R)), single-angle and 16-angle random sinograms (the worst case for
kf errors: no averaging over angles).  Run twice: RK_BP_FAN32_MAXMAG=100 (fp32 map) and =0 (fp64).
  python tools/fan_map_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402
from oracle import Geom, default_oracle, rel_l2  # noqa: E402

orc = default_oracle()
rs = np.random.default_rng(3)
out = []
for s in (96, 256):
    for target in (2.0, 3.0, 4.0, 5.0, 6.0, 8.0):
        for na in (1, 16):
            src = dd = 2.15 * s
            rmax = 0.5 * s * np.sqrt(2.0)
            sp = (src + dd) / (target * (src - rmax))
            worst = 0.0
            for trial in range(6):
                ang = list(rs.uniform(0, 2 * np.pi, na))
                g = rk.make_fanbeam(s, ang, src, dd, s, sp)
                y = rs.standard_normal((4, na, s)).astype(np.float32)
                b = rk.backprojection(g, torch.from_numpy(y).cuda()).cpu().numpy()
                rb = orc.backprojection(Geom("fanbeam", s, np.asarray(g.angles), s, sp, src, dd), y)
                worst = max(worst, rel_l2(b, rb))
            out.append((s, target, na, worst))
            print(f"s={s} mag={target:.0f} na={na} worst rel-L2 {worst:.2e}", flush=True)
