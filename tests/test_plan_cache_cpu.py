"""The on-disk forward-schedule cache (csrc/plan_cache.cpp), on host-only plans (CPU).

The reference's forward (projector.cpp:228-236) plans nothing; ours plans a
bank-conflict-aware schedule per geometry, so the second process to project
a geometry must get the same schedule (same digest = identical launches)
from the cache in milliseconds, and a stale, foreign or damaged cache file
must fall back to planning — never to a wrong schedule.
"""
import glob
import os
import time

import numpy as np
import pytest

from paper_2009_14788_b200.projector import Plan


@pytest.fixture
def cache_dir(tmp_path, monkeypatch):
    d = str(tmp_path / "plans")
    monkeypatch.setenv("RK_PLAN_CACHE", d)
    return d


def geoms(rk):
    return [rk.make_parallel(96, rk.angles_linspace(0.0, np.pi, 60)),
            rk.make_fanbeam(80, rk.angles_linspace(0.0, 2 * np.pi, 50), 100.0, det_count=97)]


def test_cache_hit_same_schedule(rk, cache_dir):
    for g in geoms(rk):
        a = Plan(g, 1.0, -1)
        ia = a.info()
        assert ia["scheduled"] and not ia["schedule_from_cache"]
        b = Plan(g, 1.0, -1)
        ib = b.info()
        assert ib["scheduled"] and ib["schedule_from_cache"]
        assert a.prepare() == b.prepare()
    assert len(glob.glob(os.path.join(cache_dir, "fwd_*.rkfs"))) == 2


def test_cache_key_covers_angles_step_and_knobs(rk, cache_dir, monkeypatch):
    g = geoms(rk)[0]
    Plan(g, 1.0, -1)
    ang = list(g.angles)
    ang[7] = np.nextafter(ang[7], 10.0)  # one bit of one angle
    assert not Plan(rk.make_parallel(96, ang), 1.0, -1).info()["schedule_from_cache"]
    assert not Plan(g, 0.75, -1).info()["schedule_from_cache"]  # step
    monkeypatch.setenv("RK_FWD_ORDER", "0")  # a planner knob
    assert not Plan(g, 1.0, -1).info()["schedule_from_cache"]


@pytest.mark.parametrize("damage", ["truncate", "flip", "garbage"])
def test_damaged_cache_file_replans(rk, cache_dir, damage):
    g = geoms(rk)[1]
    ref = Plan(g, 1.0, -1).prepare()
    (path,) = glob.glob(os.path.join(cache_dir, "fwd_*.rkfs"))
    raw = bytearray(open(path, "rb").read())
    if damage == "truncate":
        raw = raw[: len(raw) // 2]
    elif damage == "flip":  # a box record's row count (past the key): the sanity check must catch it
        raw[-9] ^= 0x7F
    else:
        raw = bytearray(b"not a schedule" * 10)
    open(path, "wb").write(bytes(raw))
    p = Plan(g, 1.0, -1)
    if damage == "flip" and p.info()["schedule_from_cache"]:
        # a flip that keeps every box inside its budget is a different but valid schedule file;
        # it can only come from a manual edit — the digest shows it differs
        assert p.prepare() != ref
    else:
        assert not p.info()["schedule_from_cache"]
        assert p.prepare() == ref


def test_disabled_cache_writes_nothing(rk, tmp_path, monkeypatch):
    monkeypatch.setenv("RK_PLAN_CACHE", "off")
    monkeypatch.setenv("HOME", str(tmp_path))
    monkeypatch.delenv("XDG_CACHE_HOME", raising=False)
    p = Plan(geoms(rk)[0], 1.0, -1)
    assert not p.info()["schedule_from_cache"]
    assert not os.path.exists(tmp_path / ".cache")


def test_warm_cache_is_fast_at_config2(rk, cache_dir):
    """cold planning vs a warm-cache plan (<= 50 ms warm)."""
    import math

    g = rk.make_parallel(512, rk.angles_linspace(0.0, math.pi, 512), 512)
    t0 = time.perf_counter()
    a = Plan(g, 1.0, -1)
    cold = time.perf_counter() - t0
    t0 = time.perf_counter()
    b = Plan(g, 1.0, -1)
    warm = time.perf_counter() - t0
    assert b.info()["schedule_from_cache"] and a.prepare() == b.prepare()
    # the warm plan still builds the fp64 ray table and backprojection windows; the schedule is read
    assert warm < 0.25 * cold, (cold, warm)


def test_concurrent_writers_publish_complete_files(rk, cache_dir):
    """Threads planning one geometry at once each write their own temporary file (plan_cache.cpp
    store_schedule) and rename it into place: every plan gets the same schedule, the published
    file loads, and no temporary file is left behind."""
    import threading

    g = rk.make_parallel(64, rk.angles_linspace(0.0, np.pi, 40))
    digests, errs = [], []

    def work():
        try:
            digests.append(Plan(g, 1.0, -1).prepare())
        except BaseException as e:  # noqa: BLE001 (re-raised below)
            errs.append(e)

    ts = [threading.Thread(target=work) for _ in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs and len(set(digests)) == 1
    assert len(glob.glob(os.path.join(cache_dir, "fwd_*.rkfs"))) == 1
    assert not glob.glob(os.path.join(cache_dir, "*.tmp.*"))
    p = Plan(g, 1.0, -1)
    assert p.info()["schedule_from_cache"] and p.prepare() == digests[0]
