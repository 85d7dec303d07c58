"""Constant ensembles: every configuration gets the same prediction, bit for
bit, in the reference's arithmetic (each hidden unit with a nonzero output
weight has zero first-layer weights on the multi-valued parameters), so the
reference's lexsort((indices, preds)) (tuner.py:110-130) returns the first m
statically valid indices. The device takes a dedicated path for them
(stats path 2: a validity scan from the slice start) instead of a guard band
that would hold every configuration (profiles/r02_band_worst_case.jsonl: 350
ms on the 10^8 space through the overflow fallback). Checked against the
oracle (which runs the reference's own lexsort) and the device's exact fp64
path."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import oracle_of_product_ensemble, oracle_space, product_space
from oracle.tuner import top_m as oracle_top_m

pytestmark = pytest.mark.gpu


def _N():
    from paper_1506_00842_b200 import _native as N
    return N


@pytest.fixture(autouse=True)
def _defaults(gpu_ok):
    N = _N()
    yield
    N.lib().mlt_ctx_set_option(N.ctx(0), N.MLT_OPT_PATH, -1)


def _ensemble(space, k=4, h=30, w1_fn=None, seed=0):
    from paper_1506_00842_b200.model import Encoder, Ensemble, Network
    rng = np.random.default_rng(seed)
    d = len(space.params)
    nets = []
    for _ in range(k):
        w1 = np.zeros((h, d)) if w1_fn is None else w1_fn(rng, h, d)
        nets.append(Network(w1, rng.uniform(-1, 1, h), rng.uniform(-1, 1, h), rng.uniform(-1, 1),
                            rng.uniform(-2, 2), rng.uniform(0.5, 2)))
    return Ensemble(nets, Encoder.from_space(space), space.name)


def _top(ens, space, m, begin=0, end=None):
    from paper_1506_00842_b200.tuner import top_m_arrays
    return top_m_arrays(ens, space, m, begin=begin, end=end, with_stats=True)


@pytest.mark.parametrize("name", ["stereo", "convolution", "raycasting"])
def test_constant_ensemble_equals_oracle_and_exact_path(name):
    N = _N()
    sp, osp = product_space(name), oracle_space(name)
    ens = _ensemble(sp)
    idx, pred, st = _top(ens, sp, 200)
    assert st["path"] == 2
    oi, op = oracle_top_m(oracle_of_product_ensemble(ens), osp, 200)
    assert np.array_equal(idx, oi)
    np.testing.assert_allclose(pred, op, rtol=1e-12, atol=0)
    assert np.all(pred == pred[0])
    N.check(N.lib().mlt_ctx_set_option(N.ctx(0), N.MLT_OPT_PATH, 1))
    ei, ep, est = _top(ens, sp, 200)
    assert est["path"] == 1
    assert np.array_equal(idx, ei)
    np.testing.assert_array_equal(pred, ep)


def test_constant_through_zero_output_weights_and_singletons():
    # units with nonzero first-layer weights but a zero output weight, and
    # weights on single-valued parameters (feature 0): still constant
    sp, osp = product_space("stereo"), oracle_space("stereo")
    single = [q for q, p in enumerate(sp.params) if len(p.values) == 1]
    ens = _ensemble(sp)
    for net in ens.members:
        net.weights_hidden[:5] = np.random.default_rng(1).uniform(-1, 1, net.weights_hidden[:5].shape)
        net.weights_out[:5] = 0.0
        for q in single:
            net.weights_hidden[:, q] = 3.0
    idx, pred, st = _top(ens, sp, 57)
    assert st["path"] == 2
    oi, op = oracle_top_m(oracle_of_product_ensemble(ens), osp, 57)
    assert np.array_equal(idx, oi)
    np.testing.assert_allclose(pred, op, rtol=1e-12, atol=0)


def test_near_constant_is_not_shortcut():
    # one tiny first-layer weight: predictions differ, so the normal paths run
    sp, osp = product_space("stereo"), oracle_space("stereo")

    def w1(rng, h, d):
        w = np.zeros((h, d))
        w[0, 0] = 1e-3
        return w
    ens = _ensemble(sp, w1_fn=w1)
    idx, pred, st = _top(ens, sp, 100)
    assert st["path"] in (0, 1)
    oi, op = oracle_top_m(oracle_of_product_ensemble(ens), osp, 100)
    assert np.array_equal(idx, oi)


def test_constant_full_1e8_space_and_slices():
    # the 10^8 space: the first m valid indices of the space / of a slice
    N = _N()
    sp, osp = product_space("synthetic-1e8"), oracle_space("synthetic-1e8")
    ens = _ensemble(sp, k=16)
    oens = oracle_of_product_ensemble(ens)
    card = sp.cardinality()
    for lo, hi, m in [(0, card, 200), (card // 8 * 3, card // 8 * 4, 200), (card - 5000, card, 4096),
                      (12345, 12345 + 3000, 50)]:
        idx, pred, st = _top(ens, sp, m, begin=lo, end=hi)
        assert st["path"] == 2
        # the oracle over a prefix of the slice long enough to hold m valid configurations
        oi, op = oracle_top_m(oens, osp, m, begin=lo, end=min(hi, lo + 4 * m + 4096))
        assert np.array_equal(idx, oi), (lo, hi, m)
        np.testing.assert_allclose(pred, op, rtol=1e-12, atol=0)
    # a sharded record (the multi-GPU step's device path) carries the same answer
    import torch
    rec = torch.empty(2 * 200 + 1, dtype=torch.int64, device="cuda")
    plan = N.plan(sp, ens, 0)
    N.check(N.lib().mlt_plan_top_m_record(plan.h, 200, 0, card, N.C.c_void_p(rec.data_ptr())))
    torch.cuda.synchronize()
    r = rec.cpu().numpy()
    full, _, _ = _top(ens, sp, 200)
    assert r[400] == 0 and np.array_equal(r[:200], full)
