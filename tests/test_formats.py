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


def test_hostile_size_fields_are_io_errors(tmp_path):
    """size fields are checked against the file length before any
    buffer is sized from them; malformed header fields / geometry are IoError
    (never a CUDA error or a crash)."""
    import struct
    import paper_2605_16360_b200 as P
    bad = str(tmp_path / "bad.pkvt")
    # header length 2^60 in a 40-byte file
    open(bad, "wb").write(b"PKVT" + struct.pack("<IQ", 1, 1 << 60) + b"L_s=1\n" * 4)
    with pytest.raises(P.TruncatedFileError, match="header"):
        P.read_trace(bad)

    def hdr(text):
        t = text.encode()
        open(bad, "wb").write(b"PKVT" + struct.pack("<IQ", 1, len(t)) + t)

    hdr("L_s=abc\nH_s=1\nL_l=1\nH_l=1\nN=4\nB=1\ndtype=f32\nsamples=0\n")
    with pytest.raises(P.IoError, match="not an integer"):
        P.read_trace(bad)
    hdr("L_s=-2\nH_s=1\nL_l=1\nH_l=1\nN=4\nB=1\ndtype=f32\nsamples=0\n")
    with pytest.raises(P.IoError, match="out of range"):
        P.read_trace(bad)
    hdr("L_s=1\nH_s=1\nL_l=1\nH_l=1\nN=4\nB=1\ndtype=f32\nsamples=-1\n")
    with pytest.raises(P.IoError, match="negative"):
        P.read_trace(bad)
    hdr("L_s=2000000000\nH_s=2000000000\nL_l=1\nH_l=1\nN=2000000000\nB=1\ndtype=f32\nsamples=1000\n")
    with pytest.raises(P.PayloadLengthError):
        P.read_trace(bad)
    # checkpoint: a tensor-name length far past the end of the file
    g = P.ModelGeometry(4, 8, 2, 4, 64)
    c = P.MapperConfig(encoder_layers=1)
    ck = str(tmp_path / "m.pkvc")
    P.write_checkpoint(ck, g, c, P.mapper_init_params(g, c, 1))
    raw = bytearray(open(ck, "rb").read())
    off = 4 + 4 + 17 * 8 + 8  # magic, version, geometry, config, tensor count
    raw[off:off + 4] = struct.pack("<I", 0xFFFFFFF0)
    open(ck, "wb").write(bytes(raw))
    with pytest.raises(P.TruncatedFileError, match="tensor name"):
        P.read_checkpoint(ck)
