"""Unusual space shapes through the device sweep: one huge parameter, many
binary parameters, single-value parameters, 32 parameters (a slice). For each,
the fp32 guard-band sweep (with and without pruning) and the fp64
materialising path must all return the ORACLE's top-m (oracle/tuner.py, the
reference's chunked predict + lexsort; ties by index included)."""

from __future__ import annotations

from functools import lru_cache

import numpy as np
import pytest

from conftest import oracle_of_product_ensemble, oracle_of_product_space

pytestmark = pytest.mark.gpu


def _space(name, radices):
    import paper_1506_00842_b200 as b
    params = tuple(b.ParamDef(f"p{i}", tuple(range(1, r + 1)) if r > 2 else ((0, 1) if r == 2 else (7,)))
                   for i, r in enumerate(radices))
    return b.ParamSpace(name, params)


def _ensemble(sp, k, scale, seed):
    import paper_1506_00842_b200 as b
    rng = np.random.default_rng(seed)
    d = len(sp.params)
    nets = [b.Network(rng.normal(size=(30, d)) * scale, rng.normal(size=30) * scale, rng.normal(size=30),
                      float(rng.normal()), float(rng.normal()), float(rng.uniform(0.2, 2))) for _ in range(k)]
    return b.Ensemble(nets, b.Encoder.from_space(sp), sp.name)


def _opt(key, value):
    from paper_1506_00842_b200 import _native as N
    N.check(N.lib().mlt_ctx_set_option(N.ctx(0), key, value))


@pytest.fixture(autouse=True)
def _reset(gpu_ok):
    from paper_1506_00842_b200 import _native as N
    yield
    for key in (N.MLT_OPT_PATH, N.MLT_OPT_PRUNE):
        N.lib().mlt_ctx_set_option(N.ctx(0), key, -1)


CASES = [
    ("one-param", [5000], None),
    ("binary20", [2] * 20, None),
    ("with-singletons", [1, 8, 1, 8, 2, 1, 16, 4, 1], None),
    ("wide-and-binary", [3000, 2, 2, 3], None),
    ("p32-slice", [2] * 32, (1 << 30, (1 << 30) + (1 << 21))),
]


@lru_cache(maxsize=None)
def _oracle_top(name, trial, m_max=100):
    """Oracle top-m_max of CASES[name] / trial (prefixes give every smaller m:
    the lexsort order is total)."""
    from oracle.tuner import top_m
    radices, rng_ = {c[0]: (c[1], c[2]) for c in CASES}[name]
    sp = _space(name, radices)
    lo, hi = rng_ if rng_ else (0, sp.cardinality())
    k, scale = [(3, 0.7), (5, 3.0)][trial]
    ens = _ensemble(sp, k, scale, 100 * len(radices) + trial)
    return top_m(oracle_of_product_ensemble(ens), oracle_of_product_space(sp), m_max, begin=lo, end=hi)


@pytest.mark.parametrize("name,radices,rng_", CASES)
@pytest.mark.parametrize("m", [1, 10, 100])
def test_band_and_pruned_equal_exact(name, radices, rng_, m):
    from paper_1506_00842_b200 import _native as N
    from paper_1506_00842_b200.tuner import top_m_arrays
    sp = _space(name, radices)
    lo, hi = rng_ if rng_ else (0, sp.cardinality())
    for trial, (k, scale) in enumerate([(3, 0.7), (5, 3.0)]):
        ens = _ensemble(sp, k, scale, 100 * len(radices) + trial)
        oi, op = _oracle_top(name, trial)
        _opt(N.MLT_OPT_PATH, 1)
        ref = top_m_arrays(ens, sp, m, begin=lo, end=hi)
        assert np.array_equal(ref[0], oi[:m]), (name, m, trial, "exact path vs oracle")
        np.testing.assert_allclose(ref[1], op[:m], rtol=1e-12, atol=0)
        _opt(N.MLT_OPT_PATH, 0)
        for prune in (0, 1):
            _opt(N.MLT_OPT_PRUNE, prune)
            got = top_m_arrays(ens, sp, m, begin=lo, end=hi, with_stats=True)
            if trial == 0:
                assert got[2]["path"] == 0, (name, got[2])        # really the fp32 guard-band sweep
            assert np.array_equal(got[0], ref[0]), (name, m, trial, prune)
            np.testing.assert_allclose(got[1], ref[1], rtol=1e-12, atol=0)
        _opt(N.MLT_OPT_PRUNE, 0)
