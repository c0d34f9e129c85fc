"""Concurrency sweep: threads on their own CUDA streams call forward / backprojection /
FBP (device and host-buffer paths) on random geometries drawn from more geometries than the
plan cache holds (LRU evictions while other threads hold plans), and every result must equal
the serial single-thread result bit for bit.
  python tools/stress_concurrency.py [threads] [iterations] [seed]"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_14788_b200 as rk  # noqa: E402

n_threads = int(sys.argv[1]) if len(sys.argv) > 1 else 8
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 40
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 0
rs = np.random.default_rng(seed)
geoms = []
for i in range(80):  # > the 64-plan LRU cache
    s = int(rs.choice([16, 24, 32, 40, 48]))
    na = int(rs.integers(4, 40))
    if i % 2:
        geoms.append(rk.make_fanbeam(s, list(rs.uniform(0, 2 * np.pi, na)), float(s) * float(rs.uniform(1.2, 3.0))))
    else:
        geoms.append(rk.make_parallel(s, list(rs.uniform(0, np.pi, na)), int(rs.integers(s // 2, 2 * s)),
                                      float(rs.uniform(0.6, 1.6))))
jobs = []
for t in range(n_threads):
    for i in range(iters):
        gi = int(rs.integers(0, len(geoms)))
        g = geoms[gi]
        B = int(rs.choice([1, 3, 4, 5, 9]))
        op = str(rs.choice(["fwd", "bp", "fbp", "fwd_host", "bp_host"]))
        shape = (B, g.image_size, g.image_size) if op.startswith("fwd") else (B, g.n_angles, g.det_count)
        x = rs.standard_normal(shape).astype(np.float32)
        jobs.append((t, gi, op, x))


def run(job):
    _, gi, op, x = job
    g = geoms[gi]
    if op == "fwd":
        return rk.forward(g, torch.from_numpy(x).cuda()).cpu().numpy()
    if op == "bp":
        return rk.backprojection(g, torch.from_numpy(x).cuda()).cpu().numpy()
    if op == "fbp":
        return rk.fbp(g, torch.from_numpy(x).cuda()).cpu().numpy()
    if op == "fwd_host":
        return np.asarray(rk.forward(g, x))
    return np.asarray(rk.backprojection(g, x))


serial = [run(j) for j in jobs]
results = [None] * len(jobs)
errors = []


def worker(t):
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for k, j in enumerate(jobs):
            if j[0] != t:
                continue
            try:
                results[k] = run(j)
            except Exception as e:  # noqa: BLE001
                errors.append((k, repr(e)))


threads = [threading.Thread(target=worker, args=(t,)) for t in range(n_threads)]
for th in threads:
    th.start()
for th in threads:
    th.join()
torch.cuda.synchronize()
bad = [k for k in range(len(jobs)) if results[k] is None or not np.array_equal(results[k], serial[k])]
for k in bad[:10]:
    print("MISMATCH job", k, jobs[k][1:3])
print(f"stress concurrency: {len(jobs)} jobs on {n_threads} threads, {len(bad)} mismatches, {len(errors)} errors "
      f"{errors[:3]}")
sys.exit(1 if bad or errors else 0)
