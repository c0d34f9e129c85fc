"""Forward-schedule invariant (CPU, host-only plans): replaying the forward
kernel's per-lane schedule in its own fp32 arithmetic, every sample's four
taps lie inside its chunk's staged box and the chunks cover every sample of
every ray (fwd_plan.cpp: verify_forward_schedule).  The kernel indexes the
box without clamping on the strength of this invariant."""
import math
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import math, sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_2009_14788_b200 as rk
rng = np.random.default_rng(7)
cases = [
    rk.make_parallel(256, rk.angles_linspace(0.0, math.pi, 256)),                      # config 1
    rk.make_parallel(512, rk.angles_linspace(0.0, math.pi, 512)),                      # config 2
    rk.make_fanbeam(512, rk.angles_linspace(0.0, 2 * math.pi, 512), 512.0),            # config 3
    rk.make_parallel(100, rk.angles_linspace(0.0, math.pi, 33), 77, 1.3),
    rk.make_parallel(64, list(rng.uniform(-10, 10, 50)), 96, 0.7),                     # scattered angles
    rk.make_parallel(96, [(i * 100.0 / 64 - 50.0) * math.pi / 180 for i in range(64)]),  # limited arc
    rk.make_fanbeam(96, rk.angles_linspace(0.0, 2 * math.pi, 64), 70.0, det_distance=300.0),  # source close
    rk.make_fanbeam(80, list(rng.uniform(0, 7, 40)), 60.0, det_distance=150.0, det_count=101),
    # coarse detectors (cells several pixels apart): the narrow-warp fallback tiers
    rk.make_fanbeam(128, rk.angles_linspace(0.0, 2 * math.pi, 40), 128.0, det_count=16),
    rk.make_fanbeam(96, rk.angles_linspace(0.0, 2 * math.pi, 24), 96.0, det_count=12),
    rk.make_parallel(128, rk.angles_linspace(0.0, math.pi, 33), 10, 14.0),
]
for i in range(30):  # random geometries: sizes, angle lists, detectors, fan distances
    s = int(rng.choice([3, 17, 40, 64, 97, 131, 200]))
    ang = list(rng.uniform(-7.0, 7.0, int(rng.integers(1, 60))))
    nd, sp = int(rng.integers(1, 3 * s + 8)), float(rng.uniform(0.3, 2.5))
    if i % 2:
        cases.append(rk.make_fanbeam(s, ang, float(s) * float(rng.uniform(0.75, 4.0)), float(rng.uniform(0.5, 3.0)) * s,
                                     nd, sp))
    else:
        cases.append(rk.make_parallel(s, ang, nd, sp))
for g in cases:
    rk.get_plan(g, None, -1)
rk.get_plan(rk.make_parallel(48, rk.angles_linspace(0.0, math.pi, 30)), rk.ProjectorOptions(0.37), -1)
print("schedules verified", len(cases) + 1)
"""


def test_forward_schedule_boxes_contain_every_sample():
    env = dict(os.environ, RK_VERIFY_PLAN="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0 and "schedules verified" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
