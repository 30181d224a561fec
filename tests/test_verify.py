"""Verify property suites (reference verify.py:17-230).

The host suites (gate, variance, covering) run here; quant / patterns / encode drive the
CUDA kernels (pkv_quantize_groups, pack/unpack, K2 k-means, the exhaustive matcher, K1-TC
and K1 through whole caches) and are GPU tests.  The analysis restatements behind the
variance and covering suites are pinned to the reference by tests/golden/analysis.npz.
"""
import dataclasses
import os

import numpy as np
import pytest

from paper_2510_05176_b200 import analysis, verify

GOLD = os.path.join(os.path.dirname(__file__), "golden", "analysis.npz")


def _all_pass(results):
    bad = [r for r in results if not r.passed]
    assert not bad, bad
    return results


def test_suite_names_and_unknown():
    assert verify.SUITE_NAMES[:5] == ("quant", "patterns", "gate", "variance", "covering")
    with pytest.raises(ValueError, match="unknown suite"):
        verify.run_suite("nope", 0)


@pytest.mark.parametrize("suite", ["gate", "variance", "covering"])
@pytest.mark.parametrize("seed", [0, 7])
def test_host_suites(suite, seed):
    res = _all_pass(verify.run_suite(suite, seed))
    assert all(r.suite == suite for r in res)


def test_failure_carries_reproducer():
    r = verify._result("quant", "x", ["seed=3 instance=5 bits=2 length=9"], 10)
    assert not r.passed and "seed=3 instance=5" in r.detail and r.detail.startswith("1 violation(s)")


def test_analysis_matches_reference_golden():
    g = np.load(GOLD, allow_pickle=False)
    for i in range(int(g["n"])):
        pts, lab, k = g[f"pts{i}"], g[f"lab{i}"], int(g[f"k{i}"])
        rep = analysis.variance_decomposition(pts, lab, k)
        assert np.array_equal(rep.total, g[f"total{i}"]) and np.array_equal(rep.intra, g[f"intra{i}"])
        assert np.array_equal(rep.inter, g[f"inter{i}"])
        cov = analysis.covering_bound_check(pts, float(g[f"rho{i}"]), 2)
        assert np.array_equal(np.array(dataclasses.astuple(cov), dtype=np.float64), g[f"cov{i}"])


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["quant", "patterns"])
def test_gpu_suites(suite):
    _all_pass(verify.run_suite(suite, 11))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [1, 2])
def test_encode_suite(seed):
    res = _all_pass(verify.run_suite("encode", seed))
    assert len(res) == 9
