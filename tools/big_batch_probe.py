"""Large batches (int64 indexing, grid limits, scratch growth): forward + backprojection of
B images at 512^2 / 512 angles, elements 0 and B-1 against the reference, and the
batched == per-element identity.  python tools/big_batch_probe.py [B]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402
from oracle import Geom, default_oracle, rel_l2  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
orc = default_oracle()
g = rk.make_parallel(512, rk.angles_linspace(0.0, np.pi, 512))
og = Geom("parallel", 512, np.asarray(g.angles), 512, 1.0)
x = torch.rand(B, 512, 512, device="cuda")
t = time.perf_counter()
y = rk.forward(g, x)
z = rk.backprojection(g, y)
torch.cuda.synchronize()
el = time.perf_counter() - t
ok = True
for e in (0, B - 1):
    xe = x[e:e + 1].cpu().numpy()
    ef = rel_l2(y[e:e + 1].cpu().numpy(), orc.forward(og, xe))
    eb = rel_l2(z[e:e + 1].cpu().numpy(), orc.backprojection(og, y[e:e + 1].cpu().numpy()))
    single = rk.forward(g, x[e:e + 1])
    same = torch.equal(single, y[e:e + 1])
    ok &= ef <= 1e-5 and eb <= 1e-5 and same
    print(f"B={B} element {e}: forward {ef:.2e} bp {eb:.2e} batched==single {same}")
print(f"big batch {B}: {'ok' if ok else 'FAIL'} ({el:.2f} s incl. first-call work)")
sys.exit(0 if ok else 1)
