"""Pin the CPU oracle (oracle/) to the real reference: every golden fixture
written by tests/golden/make_golden.py from `mltune` itself must be
reproduced — bit-exact for integer work and for the numpy arithmetic the
oracle restates operation-for-operation, to 1e-12 where a sum order may differ.
CPU only; sized to run in well under a minute."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import CASE_SPACE, golden, oracle_ensemble, oracle_space, spaces_doc, surrogates_doc


@pytest.mark.parametrize("name", ["convolution", "raycasting", "stereo", "synthetic-1e8", "conv-rules",
                                  "bench512", "tiny"])
def test_decode_mask_encode(name):
    g = golden(f"probe_{name}.npz")
    sp = oracle_space(name)
    vals = sp.decode(g["idx"])
    assert np.array_equal(vals, g["values"])
    assert np.array_equal(sp.valid_mask(vals), g["mask"])
    assert np.array_equal(sp.encode(g["idx"]), g["feat"])


def test_builtin_cardinalities():
    cards = {n: oracle_space(n).card for n in ("convolution", "raycasting", "stereo", "synthetic-1e8")}
    assert cards == {"convolution": 131072, "raycasting": 655360, "stereo": 2359296, "synthetic-1e8": 100663296}


def test_index_roundtrip():
    sp = oracle_space("stereo")
    rng = np.random.default_rng(0)
    for i in rng.integers(0, sp.card, 200).tolist():
        assert sp.index_of(sp.config_at(i)) == i


@pytest.mark.parametrize("case", list(CASE_SPACE))
def test_predictions_bit_exact(case):
    g = golden(f"pred_{case}.npz")
    ens = oracle_ensemble(case)
    assert np.array_equal(ens.predict_indices(g["idx"]), g["pred"])


@pytest.mark.parametrize("case,m", [("conv_k1", 10), ("conv_k11", 200), ("b512_k3", 600), ("b512_k3", 7)])
def test_top_m_bit_exact(case, m):
    from oracle.tuner import top_m
    g = golden(f"topm_{case}.npz")
    i, p = top_m(oracle_ensemble(case), oracle_space(CASE_SPACE[case]), m)
    assert np.array_equal(i, g[f"m{m}_i"])
    assert np.array_equal(p, g[f"m{m}_p"])


def test_top_m_sweep_cap():
    from oracle.tuner import top_m
    g = golden("topm_conv_k11.npz")
    i, p = top_m(oracle_ensemble("conv_k11"), oracle_space("convolution"), 10, sweep_cap=50_000, seed=3)
    assert np.array_equal(i, g["cap_i"]) and np.array_equal(p, g["cap_p"])


def test_top_m_rules_space():
    from oracle.model import ensemble_from_doc
    from oracle.tuner import top_m
    from conftest import model_doc
    g = golden("topm_conv-rules_k11.npz")
    i, p = top_m(ensemble_from_doc(model_doc("conv_k11")), oracle_space("conv-rules"), 10)
    assert np.array_equal(i, g["m10_i"]) and np.array_equal(p, g["m10_p"])


def test_synthetic_slice_top_m():
    from oracle.tuner import top_m
    g = golden("topm_synth_k16.npz")
    lo, hi = 98566144, 100663296
    i, p = top_m(oracle_ensemble("synth_k16"), oracle_space("synthetic-1e8"), 200, begin=lo, end=hi)
    assert np.array_equal(i, g[f"slice_{lo}_{hi}_i"]) and np.array_equal(p, g[f"slice_{lo}_{hi}_p"])


@pytest.mark.parametrize("name", ["convolution", "stereo", "synthetic-1e8", "bench512"])
def test_stage1_samples_reproduced(name):
    """sample_random + the surrogate runner (paramspace.py:223-255, measurement.py:212-258)."""
    from oracle.surrogate import OSurrogate
    g = golden(f"stage1_{name}.npz")
    sp = oracle_space(name)
    n = len(g["idx"])
    assert np.array_equal(sp.sample_indices(n, 0), g["idx"])
    t, ok = OSurrogate(surrogates_doc()[name], sp).measured_times(g["idx"], 1)
    assert np.array_equal(ok, g["ok"])
    assert np.array_equal(t[ok], g["time"][ok])


@pytest.mark.parametrize("tag", ["a", "b", "c", "d"])
def test_training_bit_exact(tag):
    from oracle.model import OTrainCfg, train
    g = golden("train_small.npz")
    sp = oracle_space("bench512")
    c = g[f"{tag}_cfg"]
    cfg = OTrainCfg(int(c[0]), float(c[1]), int(c[2]), float(c[3]), float(c[4]), int(c[5]))
    X = sp.encode(g[f"{tag}_idx"])
    y = np.log(g[f"{tag}_time"])
    nets = train(X, y, int(c[6]), cfg)
    for i, n in enumerate(nets):
        assert np.array_equal(n.W1, g[f"{tag}_{i}_W1"])
        assert np.array_equal(n.w2, g[f"{tag}_{i}_w2"])
        assert np.array_equal([n.b2, n.mean, n.std, n.first_loss, n.final_loss], g[f"{tag}_{i}_misc"])


def test_divergence_epoch():
    from oracle.model import ODivergence, OTrainCfg, fit
    g = golden("train_small.npz")
    sp = oracle_space("bench512")
    with pytest.raises(ODivergence) as e:
        fit(sp.encode(g["div_idx"]), np.log(g["div_time"]), OTrainCfg(seed=1, learning_rate=1e9, momentum=0.0), (1, 0))
    assert e.value.epoch == int(g["div_epoch"])


def test_spaces_doc_has_all_cases():
    assert set(CASE_SPACE.values()) <= set(spaces_doc())
