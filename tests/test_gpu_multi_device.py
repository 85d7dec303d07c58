"""Single-process multi-GPU top-m (`mlt_top_m_multi`, SURVEY §8(b)
`mlt_sweep_topn_multi`): shards swept concurrently by several contexts, merged
by (prediction, index). The box has one B200, so the shards' contexts share
device 0 (each context has its own stream and workspaces); the result must
equal the single-context sweep and the reference's golden top-m exactly."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import CASE_SPACE, golden, product_ensemble, product_space

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", ["conv_k11", "stereo_k8", "synth_k16", "b512_k3"])
@pytest.mark.parametrize("n_dev", [2, 3])
def test_multi_context_equals_golden(gpu_ok, case, n_dev):
    from paper_1506_00842_b200.distributed import top_m_arrays_multi_device
    from paper_1506_00842_b200.tuner import top_m_arrays
    sp, ens = product_space(CASE_SPACE[case]), product_ensemble(case)
    g = golden(f"topm_{case}.npz")
    for m in (1, 10, 200):
        key = f"m{m}_i"
        idx, pred, st = top_m_arrays_multi_device(ens, sp, m, [0] * n_dev, with_stats=True)
        ref = top_m_arrays(ens, sp, m)
        assert np.array_equal(idx, ref[0]), (case, m)
        np.testing.assert_allclose(pred, ref[1], rtol=1e-12, atol=0)
        if key in g:
            assert np.array_equal(idx, g[key]), (case, m)
        assert st["configs"] == sp.cardinality()


def test_multi_context_slices_lists_and_small_shards(gpu_ok):
    from paper_1506_00842_b200.distributed import top_m_arrays_multi_device
    from paper_1506_00842_b200.tuner import top_m_arrays
    sp, ens = product_space("convolution"), product_ensemble("conv_k11")
    card = sp.cardinality()
    rng = np.random.default_rng(5)
    for lo, hi in [(0, 5), (1000, 1003), (card - 7, card), (12345, 98765)]:
        for m in (1, 4, 50):
            got = top_m_arrays_multi_device(ens, sp, m, [0, 0, 0], begin=lo, end=hi)
            ref = top_m_arrays(ens, sp, m, begin=lo, end=hi)
            assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1]), (lo, hi, m)
    lst = np.sort(rng.choice(card, 20000, replace=False))
    for n in (0, 1, 2, 20000):
        got = top_m_arrays_multi_device(ens, sp, 30, [0, 0], indices=lst[:n])
        ref = top_m_arrays(ens, sp, 30, indices=lst[:n])
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1]), n


def test_multi_context_errors(gpu_ok):
    from paper_1506_00842_b200 import _native as N
    from paper_1506_00842_b200.distributed import top_m_arrays_multi_device
    sp, ens = product_space("bench512"), product_ensemble("b512_k3")
    with pytest.raises(ValueError):
        top_m_arrays_multi_device(ens, sp, 0, [0, 0])
    with pytest.raises(ValueError):
        top_m_arrays_multi_device(ens, sp, 5, [])
    with pytest.raises(Exception):
        top_m_arrays_multi_device(ens, sp, 5, [0, 0], begin=0, end=sp.cardinality() + 1)
    # the same context twice is refused (contexts are not re-entrant)
    c = N.ctx(0)
    arr = (N.C.c_void_p * 2)(c.value, c.value)
    ps, pe = N.packed(sp, "space"), N.packed(ens, "ensemble")
    oi, op, on = np.empty(5, np.int64), np.empty(5), N.C.c_int64()
    rc = N.lib().mlt_top_m_multi(arr, 2, N.C.byref(ps.c), N.C.byref(pe.c), 5, 0, sp.cardinality(), None, 0,
                                 N.ptr(oi, N.C.c_int64), N.ptr(op, N.C.c_double), N.C.byref(on), None)
    assert rc == N.MLT_EINVAL
    assert b"twice" in N.lib().mlt_last_error()


def test_multi_context_with_pruning_and_chunks(gpu_ok):
    """Each context may run its shard with exact pruning and chunked sweeps:
    the merged top-m is still the reference's golden list."""
    from paper_1506_00842_b200 import _native as N
    from paper_1506_00842_b200.distributed import top_m_arrays_multi_device
    sp, ens = product_space("synthetic-1e8"), product_ensemble("synth_k16")
    g = golden("topm_synth_k16.npz")
    ctxs = [N.extra_ctx(0, s) for s in range(3)]
    try:
        for c in ctxs:
            N.check(N.lib().mlt_ctx_set_option(c, N.MLT_OPT_PRUNE, 1))
            N.check(N.lib().mlt_ctx_set_option(c, N.MLT_OPT_CHUNK, 1 << 24))
        idx, pred, st = top_m_arrays_multi_device(ens, sp, 200, [0, 0, 0], with_stats=True)
        assert np.array_equal(idx, g["m200_i"])
        assert st["evaluated_frac"] < 1.0
    finally:
        for c in ctxs:
            N.lib().mlt_ctx_set_option(c, N.MLT_OPT_PRUNE, -1)
            N.lib().mlt_ctx_set_option(c, N.MLT_OPT_CHUNK, -1)
