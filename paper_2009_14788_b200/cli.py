"""Command-line front end for the hot path — the subcommands of the reference
CLI that reach it (``proj/tools/cli.cpp``): ``project``, ``backproject``,
``filter``, ``fbp``, ``solve``, ``check-adjoint``, ``bench``, ``phantom``,
``shearlet``, ``admm`` and ``png-export``, with the same
flags (angles in degrees, geometry defaults, ``--precision``), ``.npy`` files
holding the natural rank (a batch dim is lifted/squeezed like
``lift_batch``/``squeeze_batch``, cli.cpp:109-129), the same ``--json``
reports (bench schema cli.cpp:662-676) and exit codes (0 ok, 1 validation,
2 numerical; cli.cpp:718-730).  Every computation runs on the GPU.

    python -m paper_2009_14788_b200 [--json] bench --size 512 --batch 32
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

from .errors import NumericalError, ValidationError
from .npy import read_array, write_array

VERSION = "radon_b200 0.1"


def _geo_args(p, admm_names=False):
    """cli.cpp:50-74; admm_names swaps in the --n-angles / --angles-range spellings."""
    p.add_argument("--geometry", default="parallel", choices=["parallel", "fanbeam"])
    p.add_argument("--n-angles" if admm_names else "--angles", dest="angles", type=int, default=0,
                   help="projection angle count (default: from input / size)")
    p.add_argument("--angle-start", type=float, default=math.nan,
                   help="first angle in degrees (default " + ("-range/2)" if admm_names else "0)"))
    p.add_argument("--angles-range" if admm_names else "--angle-range", dest="angle_range", type=float,
                   default=math.nan, help="span in degrees (180 parallel, 360 fan)")
    p.add_argument("--det-count", type=int, default=0)
    p.add_argument("--det-spacing", type=float, default=0.0)
    p.add_argument("--source-distance", type=float, default=0.0, help="fan-beam (default: image size)")
    p.add_argument("--det-distance", type=float, default=0.0, help="fan-beam (default: source distance)")
    p.add_argument("--step", type=float, default=1.0)


def build_geometry(a, image_size, n_angles, centered=False):
    """cli.cpp:76-97 (degrees -> radians through angles_linspace); centered: the
    default start is -range/2 (admm)."""
    import paper_2009_14788_b200 as rk

    if n_angles < 1:
        raise ValidationError(f"angle count must be >= 1, got {n_angles}")
    rng = a.angle_range if not math.isnan(a.angle_range) else (360.0 if a.geometry == "fanbeam" else 180.0)
    start = a.angle_start if not math.isnan(a.angle_start) else (-rng / 2.0 if centered else 0.0)
    ang = [d * (math.pi / 180.0) for d in rk.angles_linspace(start, start + rng, n_angles)]
    dc = a.det_count if a.det_count > 0 else None
    ds = a.det_spacing if a.det_spacing > 0 else None
    if a.geometry == "fanbeam":
        src = a.source_distance if a.source_distance > 0 else float(image_size)
        dd = a.det_distance if a.det_distance > 0 else None
        return rk.make_fanbeam(image_size, ang, src, dd, dc, ds)
    return rk.make_parallel(image_size, ang, dc, ds)


def geometry_json(g):
    """cli.cpp:140-159."""
    if hasattr(g, "source_distance"):
        return {"kind": "fanbeam", "image_size": g.image_size, "n_angles": g.n_angles,
                "source_distance": g.source_distance, "det_distance": g.det_distance, "det_count": g.det_count,
                "det_spacing": g.det_spacing}
    return {"kind": "parallel", "image_size": g.image_size, "n_angles": g.n_angles, "det_count": g.det_count,
            "det_spacing": g.det_spacing}


_PREC = {"half": np.float16, "single": np.float32, "double": np.float64}


def _read(path, want):
    x = read_array(path)  # the reference's strict reader (npy.cpp:88-158)
    if x.ndim == want - 1:
        x = x[None]
    elif x.ndim != want:
        raise ValidationError(f"expected a {want - 1}-d or batched {want}-d array, got shape {x.shape}")
    return x


def _apply_precision(x, name):
    if not name:
        return x
    dt = _PREC[name]
    if dt == np.float16 and x.dtype != np.float16:
        f = x.astype(np.float32)
        h = f.astype(np.float16)
        bad = np.isinf(h) & np.isfinite(f)
        if bad.any():  # to_half_storage is checked (tensor.cpp:241-265)
            from .errors import HalfOverflowError

            i = int(np.flatnonzero(bad)[0])
            raise HalfOverflowError(f"value {float(f.flat[i])} at flat index {i} overflows half precision", i)
        return h
    return x.astype(dt)


def _write(path, x):
    write_array(path, x[0] if x.ndim >= 2 and x.shape[0] == 1 else x)  # npy.cpp:160-199


def _to_dev(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _host(t):
    return t.detach().cpu().numpy()


def main(argv=None) -> int:
    import paper_2009_14788_b200 as rk

    ap = argparse.ArgumentParser(prog="python -m paper_2009_14788_b200", description=__doc__.split("\n")[0])
    ap.add_argument("--json", action="store_true", help="emit reports as JSON on stdout")
    ap.add_argument("--version", action="version", version=VERSION)
    ap.add_argument("--threads", type=int, default=0,
                    help="cap host worker threads (planner, host copies; 0: hardware default); results do not change")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("project", help="forward-project an image to a sinogram")
    _geo_args(p)
    p.add_argument("--in", dest="inp", required=True)
    p.add_argument("-o", "--out", required=True)
    p.add_argument("--precision", choices=list(_PREC), default="")
    p = sub.add_parser("backproject", help="backproject a sinogram to an image")
    _geo_args(p)
    p.add_argument("--size", type=int, required=True)
    p.add_argument("--in", dest="inp", required=True)
    p.add_argument("-o", "--out", required=True)
    p.add_argument("--precision", choices=list(_PREC), default="")
    p = sub.add_parser("filter", help="apply a reconstruction filter to a sinogram")
    p.add_argument("--in", dest="inp", required=True)
    p.add_argument("-o", "--out", required=True)
    p.add_argument("--filter", default="ram-lak", choices=["ram-lak", "shepp-logan", "cosine", "hamming", "hann"])
    p = sub.add_parser("fbp", help="filtered backprojection reconstruction")
    _geo_args(p)
    p.add_argument("--size", type=int, required=True)
    p.add_argument("--in", dest="inp", required=True)
    p.add_argument("-o", "--out", required=True)
    p.add_argument("--filter", default="ram-lak", choices=["ram-lak", "shepp-logan", "cosine", "hamming", "hann"])
    p.add_argument("--reference", default="")
    p.add_argument("--precision", choices=list(_PREC), default="")
    p = sub.add_parser("solve", help="iterative reconstruction from a sinogram")
    _geo_args(p)
    p.add_argument("--method", required=True, choices=["landweber", "cg", "cgne"])
    p.add_argument("--iterations", type=int, default=100)
    p.add_argument("--alpha", type=float, default=0.0)
    p.add_argument("--alpha-iterations", type=int, default=20)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--tolerance", type=float, default=0.0)
    p.add_argument("--size", type=int, required=True)
    p.add_argument("--in", dest="inp", required=True)
    p.add_argument("-o", "--out", required=True)
    p.add_argument("--reference", default="")
    p.add_argument("--precision", choices=list(_PREC), default="")
    p = sub.add_parser("check-adjoint", help="dot-product test of an operator pair")
    _geo_args(p)
    p.add_argument("--operator", dest="op_name", default="projector", choices=["projector", "shearlet"])
    p.add_argument("--size", type=int, default=64)
    p.add_argument("--scales", type=int, default=5, help="shearlet scales")
    p.add_argument("--alpha", type=float, default=0.5, help="shearlet scaling exponent")
    p.add_argument("--trials", type=int, default=10)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--tolerance", type=float, default=0.0)
    p = sub.add_parser("bench", help="time forward and backprojection throughput")
    _geo_args(p)
    p.add_argument("--size", type=int, default=512)
    p.add_argument("--batch", type=int, default=1)
    p.add_argument("--precision", choices=list(_PREC), default="single")
    p.add_argument("--warmup", type=int, default=1)
    p.add_argument("--runs", type=int, default=5)
    p = sub.add_parser("phantom", help="write a Shepp-Logan head phantom")
    p.add_argument("--size", type=int, default=512)
    p.add_argument("-o", "--out", required=True)
    p.add_argument("--precision", choices=list(_PREC), default="single")
    p = sub.add_parser("shearlet", help="alpha-shearlet analysis or synthesis")
    p.add_argument("--in", dest="inp", required=True, help="input .npy (image, or coefficients with --inverse)")
    p.add_argument("-o", "--out", required=True)
    p.add_argument("--scales", type=int, default=5)
    p.add_argument("--alpha", type=float, default=0.5)
    p.add_argument("--inverse", action="store_true", help="synthesize an image from coefficients")
    p.add_argument("--cache-dir", default="", help="plan cache directory (default: RADONKIT_CACHE_DIR)")
    p = sub.add_parser("admm", help="l1-shearlet regularized reconstruction")
    _geo_args(p, admm_names=True)
    p.add_argument("--size", type=int, required=True)
    p.add_argument("--in", dest="inp", required=True)
    p.add_argument("-o", "--out", required=True)
    p.add_argument("--scales", type=int, default=5)
    p.add_argument("--alpha", type=float, default=0.5)
    p.add_argument("--p0", type=float, default=0.02)
    p.add_argument("--p1", type=float, default=0.1)
    p.add_argument("--outer", type=int, default=50)
    p.add_argument("--inner", type=int, default=50)
    p.add_argument("--progress", action="store_true", help="print the objective each outer iteration to stderr")
    p.add_argument("--cache-dir", default="")
    p.add_argument("--reference", default="")
    p = sub.add_parser("png-export", help="render an array to a 16-bit grayscale PNG")
    p.add_argument("--in", dest="inp", required=True, help="input image .npy")
    p.add_argument("-o", "--out", required=True, help="output .png path")
    p.add_argument("--lo", type=float, default=0.0, help="window low (maps to black)")
    p.add_argument("--hi", type=float, default=1.0, help="window high (maps to white)")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:  # usage errors exit 1, --help / --version 0 (cli.cpp:711-716)
        return 0 if e.code in (0, None) else 1
    if a.threads > 0:  # cli.cpp:719 set_num_threads: the host-side workers here
        import os

        import torch

        os.environ["RK_PLAN_THREADS"] = str(a.threads)
        torch.set_num_threads(a.threads)
    try:
        return _run(rk, a)
    except ValidationError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except NumericalError as e:
        print(f"numerical error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 — any other failure (missing file, I/O): exit 1 like cli.cpp:727-729
        print(f"error: {e}", file=sys.stderr)
        return 1


def _run(rk, a) -> int:
    import torch

    if a.cmd == "project":  # cli.cpp:261-273
        img = _apply_precision(_read(a.inp, 3), a.precision)
        g = build_geometry(a, img.shape[1], a.angles if a.angles > 0 else img.shape[1])
        _write(a.out, _host(rk.forward(g, _to_dev(img), rk.ProjectorOptions(a.step))))
        return 0
    if a.cmd == "backproject":  # cli.cpp:283-299
        sino = _apply_precision(_read(a.inp, 3), a.precision)
        if a.det_count == 0:
            a.det_count = sino.shape[2]
        g = build_geometry(a, a.size, a.angles if a.angles > 0 else sino.shape[1])
        _write(a.out, _host(rk.backprojection(g, _to_dev(sino), rk.ProjectorOptions(a.step))))
        return 0
    if a.cmd == "filter":  # cli.cpp:310-318
        sino = _read(a.inp, 3)
        _write(a.out, _host(rk.filter_sinogram(_to_dev(sino), rk.make_filter(a.filter, sino.shape[2]))))
        return 0
    if a.cmd == "fbp":  # cli.cpp:338-358
        sino = _apply_precision(_read(a.inp, 3), a.precision)
        if a.det_count == 0:
            a.det_count = sino.shape[2]
        g = build_geometry(a, a.size, a.angles if a.angles > 0 else sino.shape[1])
        t0 = time.perf_counter()
        rec = _host(rk.fbp(g, _to_dev(sino), a.filter))
        secs = time.perf_counter() - t0
        _write(a.out, rec)
        rep = {"command": "fbp", "filter": a.filter, "seconds": secs, "geometry": geometry_json(g), "output": a.out}
        if a.reference:
            ref = read_array(a.reference).astype(np.float64)
            rep["mse_vs_reference"] = float(np.mean((rec.reshape(ref.shape).astype(np.float64) - ref) ** 2))
        if a.json:
            print(json.dumps(rep, indent=2))
        elif a.reference:
            print(f"mse vs reference: {rep['mse_vs_reference']:.6e}")
        return 0
    if a.cmd == "solve":  # cli.cpp:397-437
        sino = _apply_precision(_read(a.inp, 3), a.precision)
        if a.det_count == 0:
            a.det_count = sino.shape[2]
        g = build_geometry(a, a.size, a.angles if a.angles > 0 else sino.shape[1])
        op = rk.projector_operator(g, rk.ProjectorOptions(a.step))
        y = _to_dev(sino)
        guess = torch.zeros((y.shape[0], a.size, a.size), dtype=y.dtype, device=y.device)
        t0 = time.perf_counter()
        alpha = None
        if a.method == "landweber":
            alpha = a.alpha if a.alpha > 0 else 0.95 * rk.estimate_alpha(op, a.alpha_iterations, a.seed)
            x = rk.landweber(op, y, guess, alpha, a.iterations)
        elif a.method == "cgne":
            x = rk.cgne(op, guess, y, a.iterations, a.tolerance)
        else:
            b = op.adjoint(y)
            x = rk.cg(lambda v: op.adjoint(op.apply(v)), guess, b, a.iterations, a.tolerance)
        rec = _host(x)
        secs = time.perf_counter() - t0
        _write(a.out, rec)
        rep = {"command": "solve", "method": a.method, "iterations": a.iterations, "seconds": secs,
               "geometry": geometry_json(g), "output": a.out}
        if alpha is not None:
            rep["alpha"] = alpha
        if a.reference:
            ref = read_array(a.reference).astype(np.float64)
            rep["mse_vs_reference"] = float(np.mean((rec.reshape(ref.shape).astype(np.float64) - ref) ** 2))
        if a.json:
            print(json.dumps(rep, indent=2))
        return 0
    if a.cmd == "check-adjoint":  # cli.cpp:581-616
        if a.trials < 1:
            raise ValidationError("--trials must be positive")
        if a.op_name == "shearlet":
            plan = rk.make_plan(a.size, a.size, [a.alpha] * a.scales)
            op = rk.shearlet_operator(plan)
            detail = {"size": a.size, "scales": a.scales, "alpha": a.alpha, "n_coeff": plan.n_coeff}
            line = f"size={a.size} scales={a.scales}"
        else:
            g = build_geometry(a, a.size, a.angles if a.angles > 0 else a.size)
            op = rk.projector_operator(g, rk.ProjectorOptions(a.step))
            detail = geometry_json(g)
            line = f"{g.__class__.__name__} size={a.size}"
        d = rk.adjoint_check(op, a.trials, a.seed)
        if a.json:
            rep = {"command": "check-adjoint", "operator": a.op_name, "defect": d, "trials": a.trials,
                   "seed": a.seed, "detail": detail}
            if a.tolerance > 0:
                rep["tolerance"] = a.tolerance
            print(json.dumps(rep, indent=2))
        else:
            print(f"adjoint defect: {d:.6e} ({a.op_name} {line} trials={a.trials} seed={a.seed})")
        if a.tolerance > 0 and not (d <= a.tolerance):
            print(f"adjoint defect {d:.6e} exceeds tolerance {a.tolerance:.6e}", file=sys.stderr)
            return 2
        return 0
    if a.cmd == "bench":  # cli.cpp:619-689 (device-timed per call, median)
        if a.runs < 5:
            raise ValidationError("--runs must be >= 5")
        g = build_geometry(a, a.size, a.angles if a.angles > 0 else a.size)
        from .phantom import shepp_logan

        one = shepp_logan(a.size)
        img = torch.from_numpy(np.repeat(one[None], a.batch, 0).astype(_PREC[a.precision])).cuda()
        opts = rk.ProjectorOptions(a.step)
        sino = rk.forward(g, img, opts)

        def time_op(fn):
            for _ in range(a.warmup):
                fn()
            runs = []
            for _ in range(a.runs):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                runs.append(e0.elapsed_time(e1))
            med = float(np.median(runs))
            return {"median_ms": med, "images_per_s": a.batch / (med / 1000.0), "runs_ms": runs}

        fwd = time_op(lambda: rk.forward(g, img, opts))
        bwd = time_op(lambda: rk.backprojection(g, sino, opts))
        rep = {"version": VERSION, "geometry": geometry_json(g), "batch": a.batch, "precision": a.precision,
               "warmup": a.warmup, "runs": a.runs, "threads": a.threads if a.threads > 0 else (os.cpu_count() or 1),
               "device": torch.cuda.get_device_name(),
               "forward": fwd, "backprojection": bwd}
        if a.json:
            print(json.dumps(rep, indent=2))
        else:
            print(f"{VERSION}\nforward: {fwd['median_ms']:.3f} ms/call median, {fwd['images_per_s']:.2f} images/s")
            print(f"backprojection: {bwd['median_ms']:.3f} ms/call median, {bwd['images_per_s']:.2f} images/s")
        return 0
    if a.cmd == "phantom":  # cli.cpp:243-251
        from .phantom import shepp_logan

        _write(a.out, shepp_logan(a.size, _PREC[a.precision]))
        return 0
    if a.cmd == "shearlet":  # cli.cpp:440-476
        if a.scales < 1:
            raise ValidationError("--scales must be positive")
        alphas = [a.alpha] * a.scales
        x = read_array(a.inp)
        if a.inverse:
            co = _lift(x, 4)
            plan = rk.make_plan_cached(co.shape[2], co.shape[3], alphas, a.cache_dir)
            if plan.n_coeff != co.shape[1]:
                raise ValidationError(f"coefficient count {co.shape[1]} does not match the plan's {plan.n_coeff}")
            _write(a.out, _host(rk.backward(plan, _to_dev(co))))
        else:
            img = _lift(x, 3)
            plan = rk.make_plan_cached(img.shape[1], img.shape[2], alphas, a.cache_dir)
            _write(a.out, _host(rk.forward(plan, _to_dev(img))))
        return 0
    if a.cmd == "admm":  # cli.cpp:478-556
        if a.scales < 1 or not (a.p0 > 0) or not (a.p1 > 0) or a.outer < 0 or a.inner < 1:
            raise ValidationError("--scales, --p0, --p1, --inner must be positive and --outer nonnegative")
        sino = _read(a.inp, 3)
        if a.det_count == 0:
            a.det_count = sino.shape[2]
        g = build_geometry(a, a.size, a.angles if a.angles > 0 else sino.shape[1], centered=True)
        op = rk.projector_operator(g, rk.ProjectorOptions(a.step))
        plan = rk.make_plan_cached(a.size, a.size, [a.alpha] * a.scales, a.cache_dir)
        y = _to_dev(sino)
        prm = rk.AdmmParams(p0=a.p0, p1=a.p1, outer_iterations=a.outer, inner_cg_iterations=a.inner)
        obs = None
        if a.progress:
            def obs(it, st):
                print(f"iter {it} objective {rk.admm_objective(op, plan, st.f, y):.6e}", file=sys.stderr)
        t0 = time.perf_counter()
        x = rk.admm_reconstruct(op, plan, y, prm, obs)
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        rec = _host(x)
        _write(a.out, rec)
        objective = rk.admm_objective(op, plan, x, y)
        rep = {"command": "admm", "outer": a.outer, "inner": a.inner, "p0": a.p0, "p1": a.p1, "scales": a.scales,
               "alpha": a.alpha, "seconds": secs, "objective": objective, "geometry": geometry_json(g),
               "output": a.out}
        if a.reference:
            ref = read_array(a.reference).astype(np.float64)
            rep["mse_vs_reference"] = float(np.mean((rec.reshape(ref.shape).astype(np.float64) - ref) ** 2))
        if a.json:
            print(json.dumps(rep, indent=2))
        else:
            print(f"admm: {a.outer} outer x {a.inner} inner iterations, objective {objective:.6e}, {secs:.3f} s")
            if a.reference:
                print(f"mse vs reference: {rep['mse_vs_reference']:.6e}")
        return 0
    if a.cmd == "png-export":  # cli.cpp:690-708
        rk.png_export(read_array(a.inp), a.out, a.lo, a.hi)
        return 0
    return 1


def _lift(x, want):
    """lift_batch (cli.cpp:109-122)."""
    if x.ndim == want - 1:
        return x[None]
    if x.ndim != want:
        raise ValidationError(f"expected a {want - 1}-d or batched {want}-d array, got shape {x.shape}")
    return x


if __name__ == "__main__":
    sys.exit(main())
