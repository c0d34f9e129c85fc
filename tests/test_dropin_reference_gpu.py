"""The reference's own program over the B200 projector.

integration/_build/dropin_check calls only the reference's public API
(projector.hpp, sino_filter.hpp, linop.hpp, solvers.hpp, npy.hpp), linked
against the reference's unmodified linop / solvers / tensor / sino_filter
code with projector_b200.cpp + sino_filter_b200.cpp in place of the
projector bodies (integration/Makefile).  Its results — forward,
backprojection, fp16 forward, FBP, filter_sinogram, and adjoint_check /
estimate_alpha / landweber / cgne from linop.cpp:65-80 and solvers.cpp:47-166
running unchanged over the GPU operator — must match the unmodified
reference (oracle/_ref) on the same inputs.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import Geom, rel_l2

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "integration", "_build", "dropin_check")


@pytest.fixture(scope="module")
def run(tmp_path_factory, cuda):
    if not os.path.exists(EXE):
        pytest.fail("integration/_build/dropin_check missing: build() makes it where /root/reference exists")
    out = tmp_path_factory.mktemp("dropin")
    r = subprocess.run([EXE, str(out)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    scalars = json.loads(r.stdout.strip().splitlines()[-1])
    return scalars, (lambda name: np.load(out / f"{name}.npy"))


@pytest.fixture(scope="module")
def ref():
    from oracle import RefOracle

    try:
        return RefOracle()
    except (FileNotFoundError, OSError):
        pytest.fail("the unmodified reference (oracle/_ref) is required as the checker here")


def par(s, na, stop=np.pi, nd=None):
    from oracle import RefOracle

    return Geom("parallel", s, RefOracle().angles_linspace(0.0, stop, na), nd)


def test_forward_backprojection_cfg2_cfg3(run, ref):
    _, load = run
    x = load("x512")
    gp = par(512, 512)
    gf = Geom("fanbeam", 512, ref.angles_linspace(0.0, 2 * np.pi, 512), source_distance=512.0)
    assert rel_l2(load("fwd_par"), ref.forward(gp, x)) <= 1e-5
    assert rel_l2(load("bp_par"), ref.backprojection(gp, load("fwd_par"))) <= 1e-5
    assert rel_l2(load("fwd_fan"), ref.forward(gf, x)) <= 1e-5
    assert rel_l2(load("bp_fan"), ref.backprojection(gf, load("fwd_fan"))) <= 1e-5
    xh = load("x512_half")
    assert xh.dtype == np.float16 and load("fwd_par_half").dtype == np.float16
    assert rel_l2(load("fwd_par_half"), ref.forward(gp, xh)) <= 1e-3


def test_fbp_and_filter(run, ref):
    _, load = run
    s1 = load("sino256")
    g1 = par(256, 256)
    assert rel_l2(load("fbp256"), ref.fbp(g1, s1)) <= 1e-5
    assert rel_l2(load("filt256_hann"), ref.filter_sinogram(s1, "hann")) <= 1e-5


def test_linop_and_solvers_unchanged_over_the_gpu_operator(run, ref):
    sc, load = run
    g5 = par(512, 256)
    gf = Geom("fanbeam", 512, ref.angles_linspace(0.0, 2 * np.pi, 512), source_distance=512.0)
    # linop.cpp:65-80 over the GPU pair reproduces the reference's own (nonzero) defect
    assert abs(sc["adjoint_defect_cfg5"] - ref.adjoint_check(g5, 1, 0)) < 1e-6
    assert abs(sc["adjoint_defect_fan512"] - ref.adjoint_check(gf, 1, 0)) < 1e-6
    ref_alpha = 0.95 * ref.estimate_alpha(g5, 20, 0)
    assert abs(sc["alpha"] - ref_alpha) <= 1e-5 * ref_alpha
    y5 = load("y5")
    z = np.zeros((1, 512, 512), np.float32)
    assert rel_l2(load("landweber10"), ref.landweber(g5, y5, z, sc["alpha"], 10)) <= 1e-5
    assert rel_l2(load("cgne10"), ref.cgne(g5, y5, z, 10)) <= 1e-3


def test_materialize_matrix(run, ref):
    _, load = run
    m = load("matrix16")
    g = par(16, 12)
    cols = ref.forward(g, np.eye(256).reshape(256, 16, 16))  # column c = forward of unit image c (double)
    assert m.shape == (12 * 16, 256)
    assert rel_l2(m, cols.reshape(256, -1).T) <= 1e-5
