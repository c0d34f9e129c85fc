import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2009_14788_b200 as rk
from oracle import Geom, default_oracle
orc = default_oracle()
for (s, ang, nd, sp, B) in [(100, [-2.8931329237874532], 35, 1.0, 12), (100, [-2.8931329237874532], 35, 1.0, 1),
                            (100, [-1.0643609229896551], 62, 0.5416597161179726, 9)]:
    g = rk.make_parallel(s, ang, nd, sp)
    rs = np.random.default_rng(0)
    y = rs.standard_normal((B, 1, nd)).astype(np.float32)
    b = rk.backprojection(g, torch.from_numpy(y).cuda()).cpu().numpy()
    rb = orc.backprojection(Geom("parallel", s, np.asarray(g.angles), nd, sp), y)
    d = np.abs(b - rb)
    bad = np.argwhere(d[0] > 1e-4)
    print("case s", s, "ang", ang, "nd", nd, "sp", sp, "B", B, "bad pixels img0:", len(bad), "max diff", d.max())
    if len(bad):
        rows = sorted(set(bad[:, 0].tolist())); cols = sorted(set(bad[:, 1].tolist()))
        print("  rows", rows[:5], "...", rows[-5:], " cols", cols[:5], "...", cols[-5:])
        i, j = bad[0]
        print("  example", (i, j), "gpu", b[0, i, j], "ref", rb[0, i, j])
        # which tile
        print("  tiles (row, col):", sorted(set((int(a) // 32, int(c) // 32) for a, c in bad)))
        th = ang[0]; c, sn = np.cos(th), np.sin(th)
        x = j - s / 2 + 0.5; yy = s / 2 - i - 0.5
        print("  kf at example", (x * c + yy * sn) / sp + nd / 2 - 0.5)
