"""Wave-quantisation paths of the sweep on the 10^8 space: the default tail
launch (last partial wave split into quarter items), whole items only
(MLT_OPT_TAIL_SPLIT = 0) and half-item CTAs (MLT_OPT_HALF_ITEMS = 1) must
return the same top-m as the exact fp64 materialising path on shards of
1/8, 1/4, 1/2 and a ragged slice, and the whole space must give the
reference's golden top-200."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, product_ensemble, product_space

pytestmark = pytest.mark.gpu


def _opt(key, val):
    from paper_1506_00842_b200 import _native as N
    N.check(N.lib().mlt_ctx_set_option(N.ctx(0), key, val))


@pytest.fixture(autouse=True)
def _restore(gpu_ok):
    yield
    from paper_1506_00842_b200 import _native as N
    for k in (N.MLT_OPT_PATH, N.MLT_OPT_TAIL_SPLIT, N.MLT_OPT_HALF_ITEMS):
        N.lib().mlt_ctx_set_option(N.ctx(0), k, -1)


@pytest.mark.parametrize("lo,hi", [(0, 100663296 // 8), (100663296 // 8 * 3, 100663296 // 8 * 4),
                                   (0, 100663296 // 4), (50331648, 100663296), (12345, 12345 + 7_000_003)])
def test_tail_modes_equal_exact_path(lo, hi):
    from paper_1506_00842_b200 import _native as N
    from paper_1506_00842_b200.tuner import top_m_arrays
    sp, ens = product_space("synthetic-1e8"), product_ensemble("synth_k16")
    _opt(N.MLT_OPT_PATH, 1)
    ref = top_m_arrays(ens, sp, 200, begin=lo, end=hi)
    _opt(N.MLT_OPT_PATH, -1)
    for tail, half in ((1, 0), (0, 0), (0, 1)):
        _opt(N.MLT_OPT_TAIL_SPLIT, tail)
        _opt(N.MLT_OPT_HALF_ITEMS, half)
        idx, pred, st = top_m_arrays(ens, sp, 200, begin=lo, end=hi, with_stats=True)
        assert st["path"] == 0
        assert np.array_equal(idx, ref[0]), (lo, hi, tail, half)
        np.testing.assert_allclose(pred, ref[1], rtol=1e-12, atol=0)


def test_tail_split_whole_space_golden():
    from paper_1506_00842_b200.tuner import top_m_arrays
    sp, ens = product_space("synthetic-1e8"), product_ensemble("synth_k16")
    g = golden("topm_synth_k16.npz")
    idx, pred = top_m_arrays(ens, sp, 200)
    assert np.array_equal(idx, g["m200_i"])
    np.testing.assert_allclose(pred, g["m200_p"], rtol=1e-12, atol=0)
