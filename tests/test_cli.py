"""The command-line front end (proj/tools/cli.cpp subcommands on the path):
argument/validation behaviour on CPU, the GPU pipeline phantom -> project ->
fbp -> solve -> check-adjoint -> bench on a B200 (test_cli.cpp:80-140, 265-291)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cli(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_2009_14788_b200", *args], capture_output=True, text=True,
                          cwd=cwd or ROOT)


def test_cli_validation_exit_codes(tmp_path):
    """cli.cpp:718-730: validation errors exit 1 (fan source inside the image)."""
    img = tmp_path / "img.npy"
    np.save(img, np.zeros((16, 16), np.float32))
    r = cli("project", "--geometry", "fanbeam", "--source-distance", "5", "--in", str(img), "-o",
            str(tmp_path / "s.npy"))
    assert r.returncode == 1 and "source_distance" in r.stderr
    r = cli("project", "--in", str(tmp_path / "missing.npy"), "-o", str(tmp_path / "s.npy"))
    assert r.returncode != 0
    r = cli("--version")
    assert r.returncode == 0 and "radon_b200" in r.stdout


@pytest.mark.gpu
def test_cli_pipeline(tmp_path, oracle, cuda):
    from paper_2009_14788_b200.phantom import shepp_logan

    ph = shepp_logan(128)
    np.save(tmp_path / "ph.npy", ph)
    assert cli("project", "--angles", "128", "--det-count", "185", "--in", str(tmp_path / "ph.npy"), "-o",
               str(tmp_path / "sino.npy")).returncode == 0
    sino = np.load(tmp_path / "sino.npy")
    assert sino.shape == (128, 185) and sino.dtype == np.float32
    r = cli("--json", "fbp", "--size", "128", "--in", str(tmp_path / "sino.npy"), "-o", str(tmp_path / "rec.npy"),
            "--reference", str(tmp_path / "ph.npy"))
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["command"] == "fbp" and rep["geometry"]["det_count"] == 185 and rep["mse_vs_reference"] < 1e-2
    r = cli("--json", "solve", "--method", "cgne", "--iterations", "20", "--size", "128", "--in",
            str(tmp_path / "sino.npy"), "-o", str(tmp_path / "cg.npy"), "--reference", str(tmp_path / "ph.npy"))
    assert r.returncode == 0, r.stderr
    assert json.loads(r.stdout)["mse_vs_reference"] < rep["mse_vs_reference"] * 5
    r = cli("--json", "check-adjoint", "--size", "64", "--angles", "90", "--trials", "10", "--tolerance", "5e-3")
    assert r.returncode == 0 and json.loads(r.stdout)["defect"] < 5e-3
    r = cli("--json", "bench", "--size", "128", "--batch", "8", "--runs", "5")
    assert r.returncode == 0, r.stderr
    b = json.loads(r.stdout)
    for key in ("version", "geometry", "batch", "precision", "warmup", "runs", "threads", "forward", "backprojection"):
        assert key in b
    assert len(b["forward"]["runs_ms"]) == 5 and b["forward"]["images_per_s"] > 0


def test_cli_phantom_matches_reference(tmp_path, ref):
    """phantom subcommand (cli.cpp:233-251) writes the reference's phantom bit for bit."""
    for prec, dt in (("single", np.float32), ("double", np.float64), ("half", np.float16)):
        r = cli("phantom", "--size", "64", "--precision", prec, "-o", str(tmp_path / f"p_{prec}.npy"))
        assert r.returncode == 0, r.stderr
        got = np.load(tmp_path / f"p_{prec}.npy")
        assert got.dtype == dt and got.shape == (64, 64)
        assert np.array_equal(got, ref.shepp_logan(64, dt)[0])


def test_npy_golden_bytes(tmp_path):
    """The .npy files the CLI writes are byte-identical to the reference's frozen
    numpy goldens (test_npy.cpp:19-35), and read back exactly (:39-71)."""
    hdr = "934e554d5059010076007b276465736372273a20273c66{}272c2027666f727472616e5f6f72646572273a2046616c73652c20"
    golden = [
        (hdr.format("34") + "277368617065273a2028322c2033292c207d" + "20" * 58 + "0a"
         "0000c03f000010c0000000000000484000009040000060bf", np.array([[1.5, -2.25, 0.0], [3.125, 4.5, -0.875]], np.float32)),
        (hdr.format("38") + "277368617065273a2028332c292c207d" + "20" * 60 + "0a"
         "9a9999999999b93f9a9999999999c9bf333333333333d33f", np.array([0.1, -0.2, 0.3], np.float64)),
        (hdr.format("32") + "277368617065273a2028322c2032292c207d" + "20" * 58 + "0a" "003c00b800340040",
         np.array([[1.0, -0.5], [0.25, 2.0]], np.float16)),
    ]
    from paper_2009_14788_b200.cli import _read, _write

    for k, (hexs, vals) in enumerate(golden):
        p = tmp_path / f"g{k}.npy"
        _write(str(p), vals)
        assert p.read_bytes() == bytes.fromhex(hexs), vals.dtype
        back = np.load(p)
        assert back.dtype == vals.dtype and np.array_equal(back, vals)
        if vals.ndim == 2:
            assert np.array_equal(_read(str(p), 3)[0], vals)


@pytest.mark.gpu
def test_cli_shearlet_and_admm(tmp_path, ref, cuda):
    """shearlet (cli.cpp:440-476) round trip and admm (cli.cpp:478-556) JSON report."""
    import math

    from paper_2009_14788_b200.phantom import shepp_logan

    ph = shepp_logan(32)
    np.save(tmp_path / "ph.npy", ph)
    r = cli("shearlet", "--scales", "3", "--in", str(tmp_path / "ph.npy"), "-o", str(tmp_path / "c.npy"))
    assert r.returncode == 0, r.stderr
    c = np.load(tmp_path / "c.npy")
    assert c.shape == (27, 32, 32)
    assert np.abs(c - ref.shearlet_forward(ph[None], [0.5] * 3)[0]).max() < 1e-5
    r = cli("shearlet", "--scales", "3", "--inverse", "--in", str(tmp_path / "c.npy"), "-o", str(tmp_path / "x.npy"))
    assert r.returncode == 0 and np.abs(np.load(tmp_path / "x.npy") - ph).max() < 1e-5
    r = cli("shearlet", "--scales", "2", "--inverse", "--in", str(tmp_path / "c.npy"), "-o", str(tmp_path / "y.npy"))
    assert r.returncode == 1 and "coefficient count" in r.stderr
    ang = [(i * 100.0 / 32 - 50.0) * math.pi / 180.0 for i in range(32)]
    import paper_2009_14788_b200 as rk
    import torch

    y = rk.forward(rk.make_parallel(32, ang), torch.from_numpy(ph[None]).cuda()).cpu().numpy()[0]
    np.save(tmp_path / "y.npy", y)
    r = cli("--json", "admm", "--size", "32", "--angles-range", "100", "--scales", "3", "--outer", "20", "--in",
            str(tmp_path / "y.npy"), "-o", str(tmp_path / "rec.npy"), "--reference", str(tmp_path / "ph.npy"))
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["command"] == "admm" and rep["outer"] == 20 and rep["mse_vs_reference"] < 1.5e-2
    assert rep["geometry"]["n_angles"] == 32


def test_cli_usage_and_io_errors_exit_1(tmp_path):
    """test_cli.cpp:197-200: unknown flags and unreadable inputs exit 1 (cli.cpp:711-729)."""
    assert cli("--no-such-flag").returncode == 1
    assert cli("project", "--in", str(tmp_path / "absent.npy"), "-o", str(tmp_path / "x.npy")).returncode == 1
    assert cli("--version").returncode == 0


@pytest.mark.gpu
def test_cli_solve_methods_reconstruct_and_report(tmp_path, cuda):
    """test_cli.cpp:111-140.  cg runs the generic CG on the normal equations and
    cgne the fused device CGNE: the same algorithm, equal to fp32 rounding (the
    reference's two paths share one implementation and agree bitwise)."""
    assert cli("phantom", "--size", "32", "-o", str(tmp_path / "ph.npy")).returncode == 0
    assert cli("project", "--in", str(tmp_path / "ph.npy"), "-o", str(tmp_path / "sino.npy"), "--angles",
               "45").returncode == 0

    def solve(method, out):
        r = cli("--json", "solve", "--method", method, "--iterations", "30", "--size", "32", "--angles", "45",
                "--in", str(tmp_path / "sino.npy"), "-o", str(tmp_path / out), "--reference", str(tmp_path / "ph.npy"))
        assert r.returncode == 0, r.stderr
        return json.loads(r.stdout)

    jl = solve("landweber", "lw.npy")
    assert jl["method"] == "landweber" and jl["alpha"] > 0.0 and jl["mse_vs_reference"] < 2e-2
    assert solve("cg", "cg.npy")["mse_vs_reference"] < 1e-2
    assert solve("cgne", "cgne.npy")["mse_vs_reference"] < 1e-2
    a, b = np.load(tmp_path / "cg.npy"), np.load(tmp_path / "cgne.npy")
    assert np.linalg.norm(a - b) <= 1e-4 * np.linalg.norm(b)


@pytest.mark.gpu
def test_cli_check_adjoint_tolerance_and_operators(cuda):
    """test_cli.cpp:161-176."""
    assert cli("check-adjoint", "--size", "32", "--trials", "5", "--tolerance", "2e-2").returncode == 0
    assert cli("check-adjoint", "--size", "32", "--trials", "5", "--tolerance", "1e-9").returncode == 2
    assert cli("check-adjoint", "--operator", "shearlet", "--size", "32", "--scales", "3", "--tolerance",
               "1e-4").returncode == 0
    r = cli("--json", "check-adjoint", "--size", "32", "--trials", "5")
    assert r.returncode == 0
    j = json.loads(r.stdout)
    assert j["operator"] == "projector" and j["trials"] == 5 and 0.0 < j["defect"] < 2e-2


@pytest.mark.gpu
def test_cli_numerical_and_validation_exit_codes(tmp_path, cuda):
    """test_cli.cpp:197-214: fan source inside the image -> 1; a diverging Landweber step -> 2."""
    assert cli("phantom", "--size", "32", "-o", str(tmp_path / "ph.npy")).returncode == 0
    assert cli("project", "--in", str(tmp_path / "ph.npy"), "-o", str(tmp_path / "sino.npy"), "--angles",
               "45").returncode == 0
    assert cli("backproject", "--size", "512", "--geometry", "fanbeam", "--source-distance", "300", "--in",
               str(tmp_path / "sino.npy"), "-o", str(tmp_path / "x.npy")).returncode == 1
    assert cli("solve", "--method", "landweber", "--alpha", "1.0", "--iterations", "60", "--size", "32", "--angles",
               "45", "--in", str(tmp_path / "sino.npy"), "-o", str(tmp_path / "x.npy")).returncode == 2


@pytest.mark.gpu
def test_cli_thread_cap_half_and_ranks(tmp_path, cuda):
    """test_cli.cpp:216-251: --threads does not change results; half precision
    flows end to end; 2-d and batched 3-d files give the same bytes."""
    assert cli("phantom", "--size", "32", "-o", str(tmp_path / "ph.npy")).returncode == 0
    assert cli("--threads", "1", "project", "--in", str(tmp_path / "ph.npy"), "-o", str(tmp_path / "s1.npy")).returncode == 0
    assert cli("--threads", "3", "project", "--in", str(tmp_path / "ph.npy"), "-o", str(tmp_path / "s3.npy")).returncode == 0
    assert (tmp_path / "s1.npy").read_bytes() == (tmp_path / "s3.npy").read_bytes()

    assert cli("phantom", "--size", "32", "-o", str(tmp_path / "ph16.npy"), "--precision", "half").returncode == 0
    assert np.load(tmp_path / "ph16.npy").dtype == np.float16
    assert cli("project", "--in", str(tmp_path / "ph16.npy"), "-o", str(tmp_path / "s16.npy")).returncode == 0
    assert np.load(tmp_path / "s16.npy").dtype == np.float16
    assert cli("fbp", "--size", "32", "--in", str(tmp_path / "s16.npy"), "-o", str(tmp_path / "rec.npy"), "--precision",
               "single").returncode == 0
    assert np.load(tmp_path / "rec.npy").dtype == np.float32

    assert cli("project", "--in", str(tmp_path / "ph.npy"), "-o", str(tmp_path / "sino2d.npy"), "--angles",
               "24").returncode == 0
    s2 = np.load(tmp_path / "sino2d.npy")
    np.save(tmp_path / "sino3d.npy", s2[None])
    for name in ("2", "3"):
        assert cli("backproject", "--size", "32", "--in", str(tmp_path / f"sino{name}d.npy"), "-o",
                   str(tmp_path / f"b{name}.npy")).returncode == 0
    assert (tmp_path / "b2.npy").read_bytes() == (tmp_path / "b3.npy").read_bytes()
