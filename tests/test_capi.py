"""CPU tests of the drop-in boundary: libpkv_b200.so loads, exports every
symbol include/*.h declares, and its host logic (retention_count, layer_pair,
window_offsets, MapperParams::init, error taxonomy) matches the reference
without a GPU. No compute calls here."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import pkv_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pkv_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    import paper_2605_16360_b200 as P
    L = P.lib()
    missing = [s for h in ("pkv_capi.h", "pkv_test_hooks.h") for s in _declared(h) if not hasattr(L, s)]
    assert not missing, missing
    assert L.pkv_abi_version() == 1
    # the Python binding covers the whole public header
    assert set(_declared("pkv_capi.h")) <= set(P._lib.SIGNATURES)


def test_no_device_means_loud_failure_not_fallback():
    import paper_2605_16360_b200 as P
    if P.lib().pkv_sm100_device_count() > 0:
        pytest.skip("a B200 is visible")
    with pytest.raises(P.NoDeviceError):
        P.Context(0)


def test_retention_count_matches_reference():
    import paper_2605_16360_b200 as P
    for rho, n in [(0.34, 3), (0.2, 32768), (0.07, 170000), (1.0, 5), (0.1, 8192), (0.5, 131072)]:
        assert P.retention_count(rho, n) == O.retention_count(rho, n)
    with pytest.raises(P.PkvValueError):
        P.retention_count(0.0, 3)
    with pytest.raises(P.PkvValueError):
        P.retention_count(1.5, 3)
    with pytest.raises(P.PkvValueError):
        P.retention_count(0.5, 0)


def test_layer_pair_and_window_offsets_match_reference():
    import paper_2605_16360_b200 as P
    g = np.load(os.path.join(ROOT, "tests", "golden", "mapper.npz"))
    for name, (ll, ls) in {"llama": (32, 16), "qwen25": (28, 24), "qwen3": (64, 28), "tiny": (4, 2)}.items():
        geo = P.ModelGeometry(ll, 8, ls, 8, 128)
        assert [P.layer_pair(l, geo) for l in range(1, ll + 1)] == g[f"pair_{name}"].tolist()
    geo = P.ModelGeometry(32, 32, 16, 32, 128)
    assert P.layer_pair(17, geo) == 9
    for bad in (0, 33):
        with pytest.raises(P.PkvValueError):
            P.layer_pair(bad, geo)
    for i in range(8):
        n, c, s = g[f"win{i}_args"].tolist()
        assert P.window_offsets(n, c, s) == g[f"win{i}_offsets"].tolist()


@pytest.mark.parametrize("kw", [{}, {"synthetic_heads": 3}, {"stage_cross": "bypass"},
                                {"stage_conv": "bypass", "stage_encoder": "bypass"}, {"encoder_layers": 0}])
def test_mapper_init_params_bit_identical_to_oracle(kw):
    import paper_2605_16360_b200 as P
    geo = P.ModelGeometry(4, 8, 2, 4, 64)
    cfg = P.MapperConfig(encoder_layers=kw.pop("encoder_layers", 2), **kw)
    blob = P.mapper_init_params(geo, cfg, 1234)
    oc = O.MapperConfig(encoder_layers=cfg.encoder_layers, **kw)
    np.testing.assert_array_equal(blob, O.mapper_init_blob(O.Geometry(4, 8, 2, 4, 64), oc, 1234))


def test_mapper_config_errors_mirror_reference():
    import paper_2605_16360_b200 as P
    geo = P.ModelGeometry(4, 8, 2, 4, 64)
    with pytest.raises(P.PkvValueError, match="stride"):
        P.mapper_init_params(geo, P.MapperConfig(crop_len=64, stride=128), 0)
    with pytest.raises(P.PkvValueError, match="divisible"):
        P.mapper_init_params(geo, P.MapperConfig(d_time=100, encoder_heads=8), 0)
    with pytest.raises(P.ConfigError):
        P.MapperConfig(stage_conv="sideways").as12()


def _run_dropin():
    import subprocess
    exe = os.path.join(ROOT, "tests", "cpp", "test_dropin")
    assert os.path.exists(exe), "build() compiles tests/cpp/test_dropin"
    return subprocess.run([exe], capture_output=True, text=True, timeout=300)


def test_cpp_dropin_header_host_logic():
    """include/proxykv_b200/proxykv.hpp: reference signatures + exception taxonomy."""
    r = _run_dropin()
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_dropin_header_on_gpu(gpu):
    r = _run_dropin()
    assert r.returncode == 0 and "gpu checks: ok" in r.stdout, r.stdout + r.stderr
