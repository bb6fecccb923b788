"""On-disk formats (formats.cpp), host-only, on CPU:
the SPEC.md:443-451 examples for the PKVT trace (round-trip equality on 3
random samples, truncated file -> truncation error naming expected vs actual
bytes, header geometry vs payload size -> length error, bad magic, version
mismatch) and the mapper checkpoint (bit-exact round trip of the
MapperParams::init blob, directory checked against the geometry/config)."""
import os

import numpy as np
import pytest

from oracle import pkv_oracle as O


def test_trace_round_trip_bit_exact(tmp_path):
    import paper_2605_16360_b200 as P
    r = np.random.RandomState(0)
    x = r.rand(3, 1, 2, 4, 300).astype(np.float32)
    y = (r.rand(3, 1, 4, 8, 300) * 7).astype(np.float32)
    y[0, 0, 0, 0, :3] = [-0.0, np.float32(1e-40), np.inf]  # signed zero, subnormal, inf survive
    p = str(tmp_path / "t.pkvt")
    P.write_trace(p, x, y, meta="generator=synthetic seed=0")
    x2, y2 = P.read_trace(p)
    assert x2.tobytes() == x.tobytes() and y2.tobytes() == y.tobytes()


def test_trace_corruptions(tmp_path):
    import paper_2605_16360_b200 as P
    x = np.ones((2, 1, 2, 4, 64), np.float32)
    y = np.zeros((2, 1, 4, 8, 64), np.float32)
    p = str(tmp_path / "t.pkvt")
    P.write_trace(p, x, y)
    raw = open(p, "rb").read()
    bad = str(tmp_path / "bad.pkvt")
    open(bad, "wb").write(raw[:-10])
    with pytest.raises(P.PayloadLengthError, match="payload is"):
        P.read_trace(bad)
    open(bad, "wb").write(raw[:10])  # cut inside the header
    with pytest.raises(P.TruncatedFileError, match=r"need \d+ bytes at offset \d+, file has \d+"):
        P.read_trace(bad)
    open(bad, "wb").write(b"XKVT" + raw[4:])
    with pytest.raises(P.BadMagicError):
        P.read_trace(bad)
    open(bad, "wb").write(raw[:4] + (7).to_bytes(4, "little") + raw[8:])
    with pytest.raises(P.VersionMismatchError):
        P.read_trace(bad)
    assert issubclass(P.TruncatedFileError, P.IoError)


def test_checkpoint_round_trip_and_layout(tmp_path):
    import paper_2605_16360_b200 as P
    geom = P.ModelGeometry(4, 8, 2, 4, 64)
    cfg = P.MapperConfig()
    blob = P.mapper_init_params(geom, cfg, 7)
    ref = O.mapper_init_blob(O.Geometry(4, 8, 2, 4, 64), O.MapperConfig(), 7)
    assert blob.tobytes() == ref.tobytes()  # MapperParams::init bit-identical
    p = str(tmp_path / "m.pkvc")
    P.write_checkpoint(p, geom, cfg, blob)
    g2, c2, b2 = P.read_checkpoint(p)
    assert g2 == geom and c2 == cfg and b2.tobytes() == blob.tobytes()
    with pytest.raises(P.PkvValueError):
        P.write_checkpoint(p, geom, cfg, blob[:-1])
    raw = open(p, "rb").read()
    open(p, "wb").write(raw[:-8])
    with pytest.raises(P.PayloadLengthError):
        P.read_checkpoint(p)
    assert os.path.getsize(p) == len(raw) - 8
