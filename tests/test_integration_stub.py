"""The reference-side ctypes binding (integration/patternkv_b200.py):
every symbol include/pkv.h declares has a prototype with the header's parameter count,
the library exports it, the struct layouts match the package's binding; on a GPU a prefill
through the stub equals the package's own (bit-exact codes)."""

import os
import re
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "integration"))
import patternkv_b200 as S  # noqa: E402


def header_decls():
    text = open(os.path.join(ROOT, "include", "pkv.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(?:int|const char\*)\s+(pkv_[a-z0-9_]+)\s*\(([^)]*)\)\s*;", text):
        params = [p for p in m.group(2).split(",") if p.strip() and p.strip() != "void"]
        out[m.group(1)] = len(params)
    return out


def test_stub_declares_every_header_symbol_with_its_arity():
    decls = header_decls()
    assert len(decls) >= 30
    assert set(decls) == set(S.SIGNATURES), set(decls) ^ set(S.SIGNATURES)
    for name, n in decls.items():
        assert len(S.SIGNATURES[name][1]) == n, name


def test_stub_loads_library_and_matches_package_binding():
    from paper_2510_05176_b200 import _lib
    lib = S.load(_lib.LIB_PATH)
    for name in S.SIGNATURES:
        assert hasattr(lib, name)
        assert len(_lib.PROTOTYPES[name][1]) == len(S.SIGNATURES[name][1]), name
    assert S.pkv_config._fields_ == _lib.PkvConfig._fields_
    assert S.pkv_cache_info._fields_ == _lib.PkvCacheInfo._fields_
    z = S.f64()
    assert lib.pkv_z_quantile(0.05, z) == 0 and abs(z.value - 1.6448536269514722) < 1e-15
    # a pointer-returning entry point keeps its 64-bit value (restype set)
    assert isinstance(lib.pkv_last_error(None), bytes)


@pytest.mark.gpu
def test_stub_prefill_matches_package():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import ctypes as C

    import paper_2510_05176_b200 as P
    from oracle import pkv_oracle as O

    U, T, d = 2, 600, 128
    ks, vs = zip(*(O.synth_unit(O.unit_seed(1, 2, u), T, d) for u in range(U)))
    k = torch.from_numpy(np.stack(ks)).cuda()
    v = torch.from_numpy(np.stack(vs)).cuda()
    cfg = P.EngineConfig(bits=2, pattern_count=16)
    codec = S.B200Codec(S.load(), P.UsageError, P.DataError)
    h = codec.create(cfg, U, d, S.PKV_F64)
    codec.prefill(h, C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()), U, T, cfg.seed)
    n = codec.info(h).committed_count
    kc = torch.empty((U, n, d), dtype=torch.uint8, device="cuda")
    vc = torch.empty_like(kc)
    codec.check(codec.lib.pkv_export_codes(h, 0, n, C.c_void_p(kc.data_ptr()), C.c_void_p(vc.data_ptr()), None))
    torch.cuda.synchronize()
    ref = P.PatternKVCache(cfg, U, d, dtype=torch.float64)
    ref.prefill(k, v)
    rk, rv = ref.codes()
    assert torch.equal(kc, rk) and torch.equal(vc, rv)
    bad = k.clone()
    bad[1, 5, 3] = float("nan")
    codec.check(codec.lib.pkv_cache_reset(h, 0, None))
    with pytest.raises(P.DataError, match="token 5, dim 3"):
        codec.prefill(h, C.c_void_p(bad.data_ptr()), C.c_void_p(v.data_ptr()), U, T, cfg.seed)
    codec.destroy(h)
