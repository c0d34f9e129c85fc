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
