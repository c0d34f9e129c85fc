"""Would per-lane sample skews cut the forward kernel's bank conflicts?  (r2 experiment)

Each lane marches its ray's samples of a chunk in a rotated order: at lockstep iteration q
lane l takes sample ms_l + (q + d_l) mod cnt_l instead of ms_l + q.  That changes which points
of neighbouring rays a quarter warp reads together (the sample stagger along the rays), a degree
of freedom the planner's layout search (orientation x pitch residue x tap order) does not have.
Per chunk: the planner's best layout, then d (0..7) per lane by coordinate descent per quarter
warp (wavefronts are charged per quarter warp, so quarters are independent), then the layout
re-picked.  Prints conflict-free-relative wavefronts before/after.
python tools/sim/lane_skew.py [n_ctas]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from conflict_model import *  # noqa: F401,F403


def chunk_lanes(ca, kb, lq, tr):
    """per chunk: (ms, cnt, a, k) of the CTA's 256 lanes (conflict_model.positions restated)."""
    a, k = cta_lanes(ca, kb, lq)
    T = np.arange(-365, 366, CH)
    out = []
    for c in range(len(T) - 1):
        Ta, Tb = T[c], T[c + 1]
        ms = np.clip(np.ceil((Ta - t0[a, k]) / h[a, k] - 0.5), 0, n[a, k]).astype(int)
        me = np.clip(np.ceil((Tb - t0[a, k]) / h[a, k] - 0.5), 0, n[a, k]).astype(int)
        cnt = me - ms
        if cnt.max() <= 0:
            continue
        out.append((ms, cnt))
    return a, k, out


def pos(a, k, ms, cnt, d, tr):
    Q = cnt.max()
    q = np.arange(Q)[:, None]
    act = q < cnt[None, :]
    rot = np.where(cnt[None, :] > 0, (q + d[None, :]) % np.maximum(cnt[None, :], 1), 0)
    m = ms[None, :] + rot
    tt = m + 0.5
    X = px0[a, k][None, :] + tt * hx[a, k][None, :]
    Y = py0[a, k][None, :] + tt * hy[a, k][None, :]
    if tr:
        X, Y = Y, X
    return np.floor(Y).astype(np.int64), np.floor(X).astype(np.int64), act


def best_layout(a, k, ms, cnt, d):
    best = None
    for tr in (0, 1):
        i, j, act = pos(a, k, ms, cnt, d, tr)
        for sw in range(3):
            for r in range(8):
                B = (np.arange(8) * r) & 7
                c = cost_chunk(i, j, act, B, sw)
                if best is None or c < best[0]:
                    best = (c, tr, sw, B)
    return best


def main():
    rng = np.random.default_rng(1)
    nct = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    ctas = [(rng.integers(0, 64), rng.integers(0, 16)) for _ in range(nct)]
    T_ide = T_base = T_skew = 0
    for ca, kb in ctas:
        lq = 0
        a, k, chunks = chunk_lanes(ca, kb, lq, 0)
        ide = base = skew = 0
        for ms, cnt in chunks:
            d = np.zeros(256, int)
            c0, tr, sw, B = best_layout(a, k, ms, cnt, d)
            ide += ideal(pos(a, k, ms, cnt, d, 0)[2])
            base += c0
            # coordinate descent on d per quarter warp (lanes 8w .. 8w+7), layout fixed
            for qw in range(32):
                sl = slice(8 * qw, 8 * qw + 8)
                if cnt[sl].max() <= 0:
                    continue

                def qcost(dd):
                    i, j, act = pos(a[sl], k[sl], ms[sl], cnt[sl], dd, tr)
                    return cost_chunk(i, j, act, B, sw)

                dq = d[sl].copy()
                cur = qcost(dq)
                for _ in range(2):
                    for p in range(1, 8):
                        for v in range(8):
                            if v == dq[p]:
                                continue
                            d2 = dq.copy()
                            d2[p] = v
                            c2 = qcost(d2)
                            if c2 < cur:
                                cur, dq = c2, d2
                d[sl] = dq
            c1 = best_layout(a, k, ms, cnt, d)[0]
            skew += c1
        T_ide += ide
        T_base += base
        T_skew += skew
        print(ca, kb, "base %.3f skew %.3f" % (base / ide, skew / ide), flush=True)
    print("TOTAL base %.3f skew %.3f" % (T_base / T_ide, T_skew / T_ide))


if __name__ == "__main__":
    main()
