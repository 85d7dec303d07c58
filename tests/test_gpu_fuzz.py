"""Randomised parity of the fp32 sweep + guard band against the oracle's
lexsort (tuner.py:110-130): random space shapes (3-9 parameters, radices
1-40, every rule kind), random ensembles (k = 1-6, weight scales from flat to
saturated), every reciprocal grouping, random m and slices, the tail-split
and whole-item launch shapes, exact pruning on and off. Index lists
bit-exact, predictions within 1e-12. Seeds are fixed, so a failure
reproduces."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _N():
    from paper_1506_00842_b200 import _native as N
    return N


@pytest.fixture(autouse=True)
def _defaults(gpu_ok):
    N = _N()
    yield
    for key in (N.MLT_OPT_GROUP, N.MLT_OPT_TAIL_SPLIT, N.MLT_OPT_PATH, N.MLT_OPT_PRUNE):
        N.lib().mlt_ctx_set_option(N.ctx(0), key, -1)


def _space(rng):
    from paper_1506_00842_b200.space import ParamDef, ParamSpace, ValidityRule
    while True:
        P = int(rng.integers(3, 10))
        radix = [int(rng.choice([1, 2, 3, 4, 5, 7, 8, 16, 40])) for _ in range(P)]
        card = int(np.prod(radix))
        if 20_000 <= card <= 400_000:
            break
    params = tuple(ParamDef(f"q{p}", tuple(int(v) for v in np.sort(rng.choice(1000, r, replace=False)) + 1))
                   for p, r in enumerate(radix))
    rules = []
    for _ in range(int(rng.integers(0, 3))):
        kind = str(rng.choice(["max-product", "max-weighted-sum", "forbidden-combination"]))
        ops = tuple(f"q{p}" for p in rng.choice(P, size=2, replace=False))
        if kind == "max-product":
            rules.append(ValidityRule(kind, ops, (1, 1), int(rng.integers(1000, 400_000))))
        elif kind == "max-weighted-sum":
            rules.append(ValidityRule(kind, ops, (int(rng.integers(1, 4)), int(rng.integers(-2, 4))),
                                      int(rng.integers(500, 3000))))
        else:
            vals = tuple(params[int(o[1:])].values[0] for o in ops)
            rules.append(ValidityRule(kind, ops, vals, 0))
    return ParamSpace("fuzz", params, tuple(rules))


def _ensemble(rng, sp):
    import paper_1506_00842_b200 as b
    k = int(rng.integers(1, 7))
    d = len(sp.params)
    scale = float(rng.choice([0.2, 1.0, 3.0, 6.0]))
    nets = [b.Network(rng.normal(size=(30, d)) * scale, rng.normal(size=30) * scale, rng.normal(size=30),
                      float(rng.normal()), float(rng.normal()), float(rng.uniform(0.2, 2))) for _ in range(k)]
    return b.Ensemble(nets, b.Encoder.from_space(sp), sp.name)


@pytest.mark.parametrize("seed", range(48))
def test_fuzz_band_path_equals_oracle(seed):
    from test_gpu_parity import _oracle_from
    from oracle.tuner import top_m as otop
    from paper_1506_00842_b200.tuner import top_m_arrays
    N = _N()
    rng = np.random.default_rng(1000 + seed)
    sp = _space(rng)
    ens = _ensemble(rng, sp)
    osp, oens = _oracle_from(sp, ens)
    card = sp.cardinality()
    c = N.ctx(0)
    N.check(N.lib().mlt_ctx_set_option(c, N.MLT_OPT_GROUP, int(rng.integers(1, 5))))
    N.check(N.lib().mlt_ctx_set_option(c, N.MLT_OPT_TAIL_SPLIT, int(rng.integers(0, 2))))
    N.check(N.lib().mlt_ctx_set_option(c, N.MLT_OPT_PRUNE, int(rng.random() < 0.4)))
    m = int(rng.choice([1, 7, 50, 200, 1000]))
    lo = int(rng.integers(0, card // 2)) if rng.random() < 0.5 else 0
    hi = int(rng.integers(lo + 1, card + 1)) if rng.random() < 0.5 else card
    oi, op = otop(oens, osp, m, begin=lo, end=hi)
    idx, pred, st = top_m_arrays(ens, sp, m, begin=lo, end=hi, with_stats=True)
    assert np.array_equal(idx, oi), (seed, st)
    np.testing.assert_allclose(pred, op, rtol=1e-12, atol=0)
