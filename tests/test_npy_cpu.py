"""The .npy contract (proj/tests/test_npy.cpp:75-240): numpy-identical bytes,
exact reads, bitwise round trips in every precision, malformed files rejected
with the field or byte offset named, atomic writes."""
import os

import numpy as np
import pytest

from paper_2009_14788_b200 import Rng, ValidationError, read_array, write_array

HDR = "934e554d5059010076007b276465736372273a20273c66{}272c2027666f727472616e5f6f72646572273a2046616c73652c20"
F32 = (HDR.format("34") + "277368617065273a2028322c2033292c207d" + "20" * 58 + "0a"
       "0000c03f000010c0000000000000484000009040000060bf")
F64 = (HDR.format("38") + "277368617065273a2028332c292c207d" + "20" * 60 + "0a"
       "9a9999999999b93f9a9999999999c9bf333333333333d33f")
F16 = HDR.format("32") + "277368617065273a2028322c2032292c207d" + "20" * 58 + "0a" "003c00b800340040"
VALS = [np.array([[1.5, -2.25, 0.0], [3.125, 4.5, -0.875]], np.float32), np.array([0.1, -0.2, 0.3], np.float64),
        np.array([[1.0, -0.5], [0.25, 2.0]], np.float16)]


@pytest.mark.parametrize("k", range(3))
def test_write_array_numpy_identical_bytes_and_exact_read(tmp_path, k):
    hexs, vals = (F32, F64, F16)[k], VALS[k]
    p = str(tmp_path / "g.npy")
    write_array(p, vals)
    assert open(p, "rb").read() == bytes.fromhex(hexs)
    np.save(str(tmp_path / "n.npy"), vals)
    assert open(str(tmp_path / "n.npy"), "rb").read() == bytes.fromhex(hexs)
    back = read_array(p)
    assert back.dtype == vals.dtype and back.shape == vals.shape and np.array_equal(back, vals)


def test_roundtrip_bitwise_every_precision(tmp_path):
    rng = Rng(42)
    for dt in (np.float16, np.float32, np.float64):
        t = rng.uniform_pm1_tensor((3, 5, 7)).astype(dt)
        p = str(tmp_path / f"rt_{np.dtype(dt).name}.npy")
        write_array(p, t)
        back = read_array(p)
        assert back.dtype == t.dtype and back.tobytes() == t.tobytes()


def _patched(hexs, old, new):
    b = bytes.fromhex(hexs)
    assert len(old) == len(new) and old.encode() in b
    return b.replace(old.encode(), new.encode())


@pytest.mark.parametrize("name,data,needle", [
    ("fortran", _patched(F32, "'fortran_order': False", "'fortran_order': True "), "fortran_order"),
    ("zerod", _patched(F64, "'shape': (3,),", "'shape': (),  "), "0-d"),
    ("empty", _patched(F32, "'shape': (2, 3)", "'shape': (3, 0)"), "empty"),
    ("int", _patched(F32, "'<f4'", "'<i4'"), "<i4"),
    ("bigendian", _patched(F32, "'<f4'", "'>f4'"), ">f4"),
    ("magic", bytes([bytes.fromhex(F32)[0] ^ 0xFF]) + bytes.fromhex(F32)[1:], "byte offset 0"),
    ("version", bytes.fromhex(F32)[:6] + b"\x02" + bytes.fromhex(F32)[7:], "byte offset 6"),
    ("truncated", bytes.fromhex(F32)[:-4], "byte offset 148"),
])
def test_read_array_rejects_malformed(tmp_path, name, data, needle):
    p = tmp_path / f"{name}.npy"
    p.write_bytes(data)
    with pytest.raises(ValidationError, match=needle.replace("(", r"\(")):
        read_array(str(p))


def test_read_missing_file_and_atomic_write(tmp_path):
    with pytest.raises(ValidationError):
        read_array(str(tmp_path / "absent.npy"))
    write_array(str(tmp_path / "out.npy"), np.array([[1.0, 2.0], [3.0, 4.0]]))
    assert os.listdir(tmp_path) == ["out.npy"]
    with pytest.raises(ValidationError):
        write_array(str(tmp_path / "no_such_dir" / "x.npy"), np.zeros(2))
