"""Generate the committed golden fixtures from the REFERENCE ITSELF.

Runs the unmodified radonkit sources compiled in place (oracle/_ref, built by
`make -C oracle ref` in the container where /root/reference exists) on small
seeded cases and stores inputs + outputs in tests/golden/golden.npz.  The
fixtures then pin the C restatement (oracle/radon_oracle.c) and the GPU
kernels on machines where the reference is absent (the GPU box).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Geom, RefOracle, batched_phantom  # noqa: E402


def main():
    R = RefOracle()
    R.set_num_threads(4)
    out = {}
    cases = {
        "par32": Geom("parallel", 32, R.angles_linspace(0.0, np.pi, 45)),
        "par48_det61_sp07": Geom("parallel", 48, R.angles_linspace(0.0, np.pi, 30), 61, 0.7),
        "fan16": Geom("fanbeam", 16, R.angles_linspace(0.0, 2 * np.pi, 24), source_distance=32.0),
        "fan40_dd90_det55": Geom("fanbeam", 40, R.angles_linspace(0.0, 2 * np.pi, 36), 55, None, 45.0, 90.0),
        "par32_step05": Geom("parallel", 32, R.angles_linspace(0.0, np.pi, 16), step=0.5),
    }
    for name, g in cases.items():
        s = g.image_size
        x = R.rng_uniform(7, 3 * s * s, True).reshape(3, s, s)
        x[1] = batched_phantom(R, s, 2)[1]
        for dt, tag in ((np.float32, "f32"), (np.float64, "f64"), (np.float16, "f16")):
            xi = x.astype(dt)
            f = R.forward(g, xi)
            b = R.backprojection(g, f)
            out[f"{name}/{tag}/image"] = xi
            out[f"{name}/{tag}/forward"] = f
            out[f"{name}/{tag}/backprojection"] = b
        out[f"{name}/angles"] = np.asarray(g.angles)
        out[f"{name}/meta"] = np.array([0 if g.kind == "parallel" else 1, s, g.n_angles,
                                        g.det_count or s, g.det_spacing or np.nan, g.source_distance,
                                        g.det_distance if g.det_distance is not None else np.nan, g.step])
    # filter + fbp
    gp = Geom("parallel", 64, R.angles_linspace(0.0, np.pi, 48), 95)
    sino = R.forward(gp, R.shepp_logan(64))
    for kind in ("ram-lak", "hann"):
        for dt, tag in ((np.float32, "f32"), (np.float16, "f16")):
            out[f"filter/{kind}/{tag}/in"] = sino.astype(dt)
            out[f"filter/{kind}/{tag}/out"] = R.filter_sinogram(sino.astype(dt), kind)
            out[f"fbp/{kind}/{tag}/out"] = R.fbp(gp, sino.astype(dt), kind)
    out["filter/angles"] = np.asarray(gp.angles)
    for kind in ("ram-lak", "shepp-logan", "cosine", "hamming", "hann"):
        for nd in (8, 95, 725):
            p, rd, rf = R.make_filter(kind, nd)
            out[f"make_filter/{kind}/{nd}/d"] = rd
            out[f"make_filter/{kind}/{nd}/f"] = rf
    # adjoint defects (linop.cpp:65-80) of the reference pair
    out["adjoint/par64_90"] = np.array(R.adjoint_check(Geom("parallel", 64, R.angles_linspace(0.0, np.pi, 90)), 10, 0))
    out["adjoint/fan64_90_D128"] = np.array(
        R.adjoint_check(Geom("fanbeam", 64, R.angles_linspace(0.0, 2 * np.pi, 90), source_distance=128.0), 10, 0))
    # rng stream
    out["rng/seed2024"] = R.rng_uniform(2024, 4096)
    out["rng/seed0_pm1"] = R.rng_uniform(0, 4096, True)
    # small Landweber / CGNE runs (solvers.cpp)
    gl = Geom("parallel", 32, R.angles_linspace(0.0, np.pi, 30))
    xs = batched_phantom(R, 32, 3)
    y = R.forward(gl, xs)
    alpha = 0.95 * R.estimate_alpha(gl, 20, 0)
    out["solver/alpha"] = np.array(alpha)
    out["solver/y"] = y
    out["solver/landweber20"] = R.landweber(gl, y, np.zeros_like(xs), alpha, 20)
    out["solver/cgne10"] = R.cgne(gl, y, np.zeros_like(xs), 10, 0.0)
    out["solver/angles"] = np.asarray(gl.angles)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print(f"wrote {len(out)} arrays to tests/golden/golden.npz")


if __name__ == "__main__":
    main()
