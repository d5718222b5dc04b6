"""ROMB basis files and the offline manifest (reference io.cpp:77-131,
test_harness.cpp:150-180, 202-217). The file functions are host code in the
library: these run without a GPU."""
import os
import struct

import numpy as np
import pytest

from paper_1602_00138_b200 import offline as O
from paper_1602_00138_b200 import romdot as R


def test_basis_files_round_trip_bit_exactly(tmp_path):  # test_harness.cpp:150-165
    V = np.zeros((5, 3), order="F")
    for i in range(15):
        V[i % 5, i // 5] = np.sqrt(2.0) * (i - 7)
    markers = [O.COL_EIGENVECTOR, O.COL_INITIAL_SOLUTION, O.COL_CORRECTION]
    path = tmp_path / "v.romb"
    R.romb_write(path, V, markers)
    V2, m2 = R.romb_read(path)
    assert V2.shape == (5, 3)
    assert V2.tobytes(order="F") == V.tobytes(order="F")
    assert list(m2) == markers
    with pytest.raises(R.IoError):
        R.romb_read(tmp_path / "missing.romb")
    with pytest.raises(R.IoError):
        R.romb_write(path, V, [0, 1])


def test_version1_layout_is_the_reference_format(tmp_path):
    """A float64 basis is written as io.cpp:77-91 lays it out, byte for byte,
    and a file built from that layout by hand reads back."""
    rng = np.random.default_rng(3)
    V = np.asfortranarray(rng.standard_normal((7, 4)))
    mk = np.array([0, 0, 1, 2], dtype=np.uint8)
    ref = b"ROMB" + struct.pack("<IQQ", 1, 7, 4) + V.tobytes(order="F") + mk.tobytes()
    path = tmp_path / "ours.romb"
    R.romb_write(path, V, mk)
    assert path.read_bytes() == ref
    (tmp_path / "theirs.romb").write_bytes(ref)
    V2, m2 = R.romb_read(tmp_path / "theirs.romb")
    assert np.array_equal(V2, V) and np.array_equal(m2, mk)


def test_complex_basis_uses_version2_with_dtype_byte(tmp_path):
    rng = np.random.default_rng(4)
    V = np.asfortranarray(rng.standard_normal((6, 3)) + 1j * rng.standard_normal((6, 3)))
    path = tmp_path / "c.romb"
    R.romb_write(path, V, [2, 2, 2])
    raw = path.read_bytes()
    assert raw[:4] == b"ROMB" and struct.unpack("<IQQB", raw[4:25]) == (2, 6, 3, 1)
    assert R.romb_info(path) == (np.complex128, 6, 3)
    V2, m2 = R.romb_read(path)
    assert V2.dtype == np.complex128 and V2.tobytes(order="F") == V.tobytes(order="F")


def test_bad_files_are_io_errors(tmp_path):
    V = np.ones((4, 2), order="F")
    good = tmp_path / "g.romb"
    R.romb_write(good, V, [0, 1])
    raw = good.read_bytes()
    (tmp_path / "magic.romb").write_bytes(b"XXXX" + raw[4:])
    (tmp_path / "ver.romb").write_bytes(raw[:4] + struct.pack("<I", 7) + raw[8:])
    (tmp_path / "trunc.romb").write_bytes(raw[:-5])
    for name, msg in (("magic", "not a basis file"), ("ver", "unsupported"), ("trunc", "truncated")):
        with pytest.raises(R.IoError, match=msg):
            R.romb_read(tmp_path / f"{name}.romb")


def test_manifest_round_trip_and_sci_format(tmp_path):  # test_harness.cpp:167-180
    path = str(tmp_path / "m.txt")
    O.write_manifest(path, {"hash": "abc", "n": "42"})
    m = O.read_manifest(path)
    assert m["hash"] == "abc" and m["n"] == "42"
    assert O.format_sci(12345.678) == "1.23457e+04"
    assert O.format_sci(-1e-9) == "-1.00000e-09"
    with open(path, "a") as f:
        f.write("# comment\n\nbroken line\n")
    with pytest.raises(R.IoError, match="malformed"):
        O.read_manifest(path)


def test_config_hash_depends_on_the_seed_defining_fields():
    from paper_1602_00138_b200 import problem as P
    import dataclasses
    c = P.CONFIGS["T3"]
    assert O.config_hash(c) == O.config_hash(P.CONFIGS["T3"])
    assert O.config_hash(c) != O.config_hash(dataclasses.replace(c, k=c.k + 1))
    assert O.config_hash(c) != O.config_hash(dataclasses.replace(c, seed=c.seed + 1))
