"""Host-side logic of the product package (no GPU): the API mirror of the
reference (spaces, configs, sampling stream, RNG draw order of training,
persistence, validation errors) checked against the oracle and fixtures."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import golden, model_doc, oracle_space, product_space, spaces_doc


def test_builtin_spaces_match_reference_definitions():
    import paper_1506_00842_b200 as b
    from paper_1506_00842_b200.space import space_to_json
    for name in b.BUILTIN_SPACE_NAMES:
        assert space_to_json(b.builtin_space(name)) == spaces_doc()[name]


def test_config_index_roundtrip_and_validation():
    import paper_1506_00842_b200 as b
    sp = product_space("stereo")
    osp = oracle_space("stereo")
    for i in (0, 1, 12345, sp.cardinality() - 1):
        assert sp.config_at(i) == osp.config_at(i)
        assert sp.index_of(sp.config_at(i)) == i
    with pytest.raises(b.ConfigMismatchError):
        sp.index_of((1, 2))
    with pytest.raises(IndexError):
        sp.config_at(sp.cardinality())


@pytest.mark.parametrize("name", ["convolution", "synthetic-1e8"])
def test_sampling_stream_matches_reference(name):
    g = golden(f"stage1_{name}.npz")
    assert np.array_equal(product_space(name).sample_indices(len(g["idx"]), 0), g["idx"])


def test_rule_scalar_semantics_wrap_like_numpy():
    from paper_1506_00842_b200.space import ValidityRule
    g = golden("probe_conv-rules.npz")
    sp = product_space("conv-rules")
    for row, ok in zip(g["values"][:300], g["mask"][:300]):
        assert sp.is_statically_valid(tuple(int(v) for v in row)) == bool(ok)
    r = ValidityRule("max-weighted-sum", ("a", "b"), (1, -64), bound=0)
    assert r.is_satisfied({"a": 10, "b": 1})


def test_training_rng_draw_order_matches_reference():
    """The host draws W1, then w2, then one permutation per epoch from
    PCG64(SeedSequence([seed, member])) exactly as model.py:204-218."""
    from oracle.space import make_rng
    from paper_1506_00842_b200.model import TrainConfig, _member_draws
    cfg = TrainConfig(epochs=3, seed=9, weight_init_scale=0.7)
    w1, w2, perms = _member_draws(50, 5, cfg, (9, 2))
    rng = make_rng(9, 2)
    assert np.array_equal(w1, rng.uniform(-0.5, 0.5, (30, 5)) * 0.7)
    assert np.array_equal(w2, rng.uniform(-0.5, 0.5, 30) * 0.7)
    for e in range(3):
        assert np.array_equal(perms[e], rng.permutation(50))


def test_fold_rows_match_reference():
    from oracle.model import fold_rows
    from paper_1506_00842_b200.space import make_rng
    n, k, seed = 1663, 11, 0
    folds = np.array_split(make_rng(seed).permutation(n), k)
    mine = [np.setdiff1d(np.arange(n), f, assume_unique=True) for f in folds]
    for a, b in zip(mine, fold_rows(n, k, seed)):
        assert np.array_equal(a, b)
    sizes = sorted(len(r) for r in mine)
    assert sizes[-1] - sizes[0] <= 1


def test_model_json_roundtrip_is_lossless(tmp_path):
    from paper_1506_00842_b200.model import load_model, model_from_json, model_to_json, save_model
    ens = model_from_json(model_doc("stereo_k8"))
    save_model(ens, tmp_path / "m.json")
    back = load_model(tmp_path / "m.json")
    for a, b in zip(ens.members, back.members):
        assert np.array_equal(a.weights_hidden, b.weights_hidden)
        assert a.bias_out == b.bias_out and a.target_std == b.target_std
    assert json.loads((tmp_path / "m.json").read_text()) == json.loads(json.dumps(model_to_json(ens)))


def test_model_json_is_the_reference_schema():
    """A reference-written model file loads, and re-serialises to the same document."""
    from paper_1506_00842_b200.model import model_from_json, model_to_json
    doc = model_doc("conv_k11")
    assert json.loads(json.dumps(model_to_json(model_from_json(doc)))) == doc


def test_parse_errors(tmp_path):
    import paper_1506_00842_b200 as b
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(b.ParseError):
        b.load_model(tmp_path / "bad.json")
    with pytest.raises(b.ParseError):
        b.load_space(tmp_path / "bad.json")


def test_config_validation():
    import paper_1506_00842_b200 as b
    with pytest.raises(ValueError):
        b.TrainConfig(epochs=0)
    with pytest.raises(ValueError):
        b.TrainConfig(momentum=1.0)
    with pytest.raises(ValueError):
        b.TunerConfig(n_train=5, m_candidates=1, k_bag=11)
    with pytest.raises(ValueError):
        b.TunerConfig(n_train=50, m_candidates=0)
    with pytest.raises(ValueError):
        b.top_m_predicted(None, product_space("tiny"), 0)


def test_measure_configs_short_circuits_static_invalids():
    import paper_1506_00842_b200 as b

    class Spy:
        default_repetitions = 3
        seen = []

        def measure(self, config, repetitions=None):
            self.seen.append(config)
            return b.Sample(config, b.Outcome.valid(1.0))

    sp = b.ParamSpace("r", (b.ParamDef("a", (1, 2)), b.ParamDef("b", (1, 2))),
                      (b.ValidityRule("max-product", ("a", "b"), bound=2),))
    spy = Spy()
    out = b.measure_configs(sp, spy, [(1, 1), (2, 2), (1, 2)])
    assert [s.outcome.status for s in out] == ["valid", "invalid-static", "valid"]
    assert spy.seen == [(1, 1), (1, 2)] and out[1].repetitions == 3


def test_install_rebinds_a_reference_shaped_package():
    """install() swaps the module globals autotune resolves (tuner.py:25,152,155)."""
    import types
    import paper_1506_00842_b200 as b
    fake = types.ModuleType("fakemltune")
    fake.tuner = types.ModuleType("fakemltune.tuner")
    fake.evaluation = types.ModuleType("fakemltune.evaluation")
    errs = types.ModuleType("fakemltune.errors")
    for n in ("ConfigMismatchError", "InsufficientDataError", "DivergenceError", "EmptySpaceError",
              "AllCandidatesInvalidError"):
        setattr(errs, n, type(n, (Exception,), {}))
    import sys
    sys.modules["fakemltune.errors"] = errs
    fake.tuner.top_m_predicted = fake.tuner.train_ensemble = fake.evaluation.train_ensemble = None
    fake.top_m_predicted = fake.train_ensemble = None
    try:
        b.install(fake)
        assert fake.tuner.top_m_predicted is b.top_m_predicted
        assert fake.evaluation.train_ensemble is b.train_ensemble
        from paper_1506_00842_b200 import errors
        assert errors.active["DivergenceError"] is errs.DivergenceError
    finally:
        b.uninstall()
        del sys.modules["fakemltune.errors"]
    assert fake.tuner.top_m_predicted is None


def test_surrogate_spec_packing():
    """The mlt_surrogate descriptor built from the reference's spec JSON
    (measurement.py:497-554): term positions/values/factors in spec order,
    launch rules in the mlt_space encoding, log_sigma as SurrogateSpec computes it."""
    from conftest import surrogates_doc
    from paper_1506_00842_b200.surrogate import PackedSurrogate
    doc = surrogates_doc()["synthetic-1e8"]
    sp = product_space("synthetic-1e8")
    pk = PackedSurrogate(doc, sp)
    names = sp.param_names()
    assert pk.c.n_terms == len(doc["terms"]) and pk.c.n_rules == len(doc["invalid_rules"])
    for t, term in enumerate(doc["terms"]):
        assert pk.nparams[t] == len(term["params"])
        assert [names[p] for p in pk.tpos[t, :len(term["params"])]] == term["params"]
        assert list(pk.match[t, :len(term["match"])]) == term["match"]
        assert pk.factor[t] == term["factor"]
    assert pk.log_sigma == float(np.sqrt(np.log1p(doc["noise_cv"] ** 2)))
    assert pk.c.seed == doc["seed"] and pk.c.base_time == doc["base_time"]
    assert list(pk.kind[:pk.c.n_rules]) == [0] * pk.c.n_rules      # gpu-a: max-product launch limits
    noiseless = PackedSurrogate(dict(doc, noise_cv=0.0), sp)
    assert noiseless.c.log_sigma == 0.0


@pytest.mark.parametrize("name", ["bench512", "synthetic-1e8"])
def test_iter_random_indices_prefix_stable(name):
    """paramspace.py:237-255: the stream equals sample_indices' draw (permutation
    below 2^22 configurations, rejection sampling above) and is prefix-stable."""
    import itertools
    sp = product_space(name)
    head = list(itertools.islice(sp.iter_random_indices(17), 300))
    assert head == sp.sample_indices(300, 17).tolist()
    assert list(itertools.islice(sp.iter_random_indices(17), 120)) == head[:120]
    assert len(set(head)) == 300


def test_configs_at_matches_config_at():
    """The column-wise decode equals config_at (paramspace.py:184-193) on every
    golden space, on a 62-binary-parameter space and past int64 values."""
    import paper_1506_00842_b200 as b
    rng = np.random.default_rng(3)
    spaces = [product_space(n) for n in ("bench512", "synthetic-1e8", "convolution", "stereo", "raycasting")]
    spaces.append(b.ParamSpace("p62", tuple(b.ParamDef(f"p{i}", (0, 1)) for i in range(62))))
    spaces.append(b.ParamSpace("huge-values", (b.ParamDef("a", (1, 2 ** 70)), b.ParamDef("b", (3, 4, 5)))))
    for sp in spaces:
        card = sp.cardinality()
        idx = np.unique(np.concatenate([rng.integers(0, card, 64), [0, card - 1]]))
        got = sp.configs_at(idx)
        assert got == [sp.config_at(int(i)) for i in idx], sp.name
        assert all(type(v) is int for v in got[0])
    assert spaces[0].configs_at([]) == []
    with pytest.raises(IndexError):
        spaces[0].configs_at([spaces[0].cardinality()])
