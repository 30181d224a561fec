"""CPU checks of the C ABI (no GPU compute): the library loads, exports every
symbol include/pkv.h declares, the host-side gate constants equal the
reference's golden values, config validation follows the reference error
taxonomy, and cache creation fails loudly without a device."""

import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "pkv.h")).read()
    return sorted(set(re.findall(r"\b(pkv_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2510_05176_b200 import _lib

    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(_lib.load(), s), s
        assert s in _lib.PROTOTYPES, f"{s} has no ctypes prototype"


def test_gate_constants_match_reference_golden():
    import paper_2510_05176_b200 as P

    g = np.load(os.path.join(ROOT, "tests", "golden", "gate.npz"))
    for j, a in enumerate(g["alphas"]):
        assert P.z_quantile(float(a)) == g["z"][j]
        for i, d in enumerate(g["dims"]):
            want = g["thr"][i, j]
            if np.isnan(want):
                with pytest.raises(P.UsageError):
                    P.contraction_threshold(int(d), float(a))
            else:
                assert P.contraction_threshold(int(d), float(a)) == want
    assert P.contraction_threshold(128, 0.05) == 0.9115533837525618


def test_decide_semantics():
    import math

    import paper_2510_05176_b200 as P

    gate = P.GateConfig.create(128, 0.05)
    assert P.decide(10.0, 9.0, gate).flatten  # test_gate.py:122-126
    d = P.decide(0.0, 1.0, gate)
    assert not d.flatten and d.ratio == math.inf
    with pytest.raises(P.UsageError):
        P.decide(-1.0, 0.0, gate)
    m, v = P.expected_error_gain(3.0, 0.0, 2, 4)
    assert m == pytest.approx(1 / 12) and v == pytest.approx(1 / 720)


def test_config_validation_taxonomy():
    import paper_2510_05176_b200 as P

    cfg = P.EngineConfig()
    assert (cfg.bits, cfg.pattern_count, cfg.group_size, cfg.residual_window) == (2, 32, 128, 128)
    assert cfg.use_k_patterns and cfg.use_v_patterns and cfg.generate_new_patterns and cfg.use_v_gate
    assert not cfg.use_k_gate
    for bad in (dict(bits=3), dict(pattern_count=0), dict(group_size=0), dict(group_size=64, residual_window=32),
                dict(alpha=0.0)):
        with pytest.raises(P.UsageError):
            P.EngineConfig(**bad)
    raw = P.EngineConfig(bits=4, group_size=64, residual_window=64).raw_variant()
    assert raw.is_raw and raw.bits == 4 and raw.group_size == 64


def test_bits_per_token_closed_form():
    import paper_2510_05176_b200 as P

    cfg = P.EngineConfig(bits=2, pattern_count=32)
    assert P.bits_per_token(cfg, 128, 32, 4096, "v") == 320.0  # test_acceptance.py:469-470
    assert P.fp16_reference_bits_per_token(128) == 2048.0


def test_no_device_fails_loudly():
    import torch

    import paper_2510_05176_b200 as P

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(P.UsageError, match="no CPU fallback"):
        P.PatternKVCache(P.EngineConfig(), 1, 128)
    with pytest.raises(P.UsageError):
        P.quantize_group(np.array([0.0, 1.0]), 2)
    # the C ABI itself refuses too
    from paper_2510_05176_b200 import _lib
    from paper_2510_05176_b200.cache import make_config_struct

    h = C.c_void_p()
    s = make_config_struct(P.EngineConfig())
    rc = _lib.load().pkv_cache_create(C.byref(s), 1, 128, _lib.PKV_F16, 1024, 64, 0, C.byref(h))
    assert rc == _lib.PKV_USAGE
    assert "no CUDA device" in _lib.last_error()[0]


def test_import_fails_loudly_without_library_and_build_module_runs_from_clean_tree():
    """No CPU fallback: importing the package without libpkv_b200.so raises ImportError;
    `python -m paper_2510_05176_b200.build` does not need the library to exist."""
    import subprocess
    import sys

    env = dict(os.environ, PKV_LIB="/nonexistent/libpkv_b200.so")
    r = subprocess.run([sys.executable, "-c", "import paper_2510_05176_b200"], cwd=ROOT, env=env,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "ImportError" in r.stderr and "no CPU fallback" in r.stderr
    # the package __init__ skips the eager load only for the build module run as __main__
    r = subprocess.run([sys.executable, "-c", "import sys; sys.orig_argv = ['python', '-m', "
                        "'paper_2510_05176_b200.build']; import paper_2510_05176_b200; print('ok')"],
                       cwd=ROOT, env=env, capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr
