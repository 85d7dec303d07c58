"""The reference's own behavioural pins for this path (SURVEY §8(c) list),
re-run against the device implementation: the same spaces, surrogates, seeds
and assertions as /root/reference/pkg/tests/test_model.py and
test_paramspace.py, with every numeric call going through the sm_100a
library (training `k_train`, prediction `k_predict64`, decode / masks
`k_decode` / `k_valid`, measurements `k_surr_times`)."""

from __future__ import annotations

import itertools
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _b():
    import paper_1506_00842_b200 as b
    return b


def _tiny():
    b = _b()
    return b.ParamSpace("tiny", (b.ParamDef("a", (1, 2, 4)), b.ParamDef("b", (0, 1)),
                                 b.ParamDef("c", (10, 20, 30, 40))))


def _space512():
    b = _b()
    return b.ParamSpace("bench512", (
        b.ParamDef("wg_x", (1, 2, 4, 8, 16, 32, 64, 128)),
        b.ParamDef("ppt_x", (1, 2, 4, 8, 16, 32, 64, 128)),
        b.ParamDef("flag_a", (0, 1)), b.ParamDef("flag_b", (0, 1)), b.ParamDef("flag_c", (0, 1))))


def _surrogate512():
    """conftest.make_surrogate512 (seed 11), noise-free as in _make_training_case:
    the spec the committed eval fixture carries, with noise_cv = 0."""
    import dataclasses
    import json
    from conftest import GOLDEN
    from paper_1506_00842_b200.formats import surrogate_from_json
    spec = surrogate_from_json(json.loads((GOLDEN / "eval_bench512.json").read_text())["surrogate"])
    return dataclasses.replace(spec, noise_cv=0.0)


def _collect(space, runner, n, seed):
    """conftest.collect_samples: the seeded sample, measured (tests/conftest.py:23-26)."""
    b = _b()
    return b.SampleSet(space, getattr(runner, "runner_id", "runner"),
                       tuple(b.measure_configs(space, runner, space.sample_random(n, seed))))


def _training_case(n=200, seed=6):
    sp = _space512()
    return sp, _collect(sp, _b().B200SurrogateRunner(_surrogate512(), sp), n, seed)


def _const_net(log_time, dim):
    return _b().Network(np.zeros((30, dim)), np.zeros(30), np.zeros(30), log_time)


# ---- test_model.py ------------------------------------------------------------------

def test_single_sample_memorized(gpu_ok):
    """test_model.py:208-213."""
    b = _b()
    sp = b.ParamSpace("one", (b.ParamDef("x", (0, 1)),))
    ss = b.SampleSet(sp, "r", (b.Sample((1,), b.Outcome.valid(2.0)),))
    net = b.train_network(ss, sp, b.TrainConfig(seed=1))
    got = float(net.predict_log_batch(b.Encoder.from_space(sp).encode((1,))[np.newaxis, :])[0])
    assert abs(got - math.log(2.0)) <= 0.01 * abs(math.log(2.0))


def test_two_level_surrogate_recovered_within_five_percent(gpu_ok):
    """test_model.py:216-230."""
    b = _b()
    from paper_1506_00842_b200.formats import SurrogateSpec, SurrogateTerm
    sp = b.ParamSpace("lvl", (b.ParamDef("flag", (0, 1)), b.ParamDef("d1", (0, 1)), b.ParamDef("d2", (0, 1, 2))))
    spec = SurrogateSpec(base_time=1.0, terms=(SurrogateTerm(("flag",), (1,), 0.5),))
    ss = _collect(sp, b.B200SurrogateRunner(spec, sp), 10, 4)
    ens = b.train_ensemble(ss, sp, k=1, cfg=b.TrainConfig(seed=2))
    for i in range(sp.cardinality()):
        cfg = sp.config_at(i)
        assert b.predict(ens, cfg) == pytest.approx(0.5 if cfg[0] == 1 else 1.0, rel=0.05)


def test_training_is_deterministic(gpu_ok):
    """test_model.py:233-241: identical inputs give bitwise-identical weights."""
    b = _b()
    sp, ss = _training_case()
    cfg = b.TrainConfig(seed=9, epochs=40)
    x, y = b.train_network(ss, sp, cfg), b.train_network(ss, sp, cfg)
    assert np.array_equal(x.weights_hidden, y.weights_hidden)
    assert np.array_equal(x.biases_hidden, y.biases_hidden)
    assert np.array_equal(x.weights_out, y.weights_out)
    assert x.bias_out == y.bias_out


def test_training_loss_decreases(gpu_ok):
    """test_model.py:261-264."""
    b = _b()
    sp, ss = _training_case()
    net = b.train_network(ss, sp, b.TrainConfig(seed=3))
    assert net.final_epoch_loss < net.first_epoch_loss


def test_invalid_only_and_too_few_samples(gpu_ok):
    """test_model.py:244-255, :276-279."""
    b = _b()
    sp = _tiny()
    ss = b.SampleSet(sp, "r", (b.Sample(sp.config_at(0), b.Outcome.invalid("invalid-launch")),
                               b.Sample(sp.config_at(1), b.Outcome.invalid("invalid-static"))))
    with pytest.raises(b.InsufficientDataError):
        b.train_network(ss, sp, b.TrainConfig())
    with pytest.raises(b.InsufficientDataError):
        b.train_ensemble(ss, sp, k=1)
    sp512, few = _training_case(n=8)
    with pytest.raises(b.InsufficientDataError):
        b.train_ensemble(few, sp512, k=11)


def test_k1_ensemble_equals_single_network(gpu_ok):
    """test_model.py:283-292."""
    b = _b()
    sp, ss = _training_case(n=100)
    cfg = b.TrainConfig(seed=5, epochs=60)
    single = b.train_network(ss, sp, cfg)
    ens = b.train_ensemble(ss, sp, k=1, cfg=cfg)
    assert np.array_equal(ens.members[0].weights_hidden, single.weights_hidden)
    config = sp.config_at(17)
    log_single = float(single.predict_log_batch(b.Encoder.from_space(sp).encode(config)[np.newaxis, :])[0])
    assert b.predict(ens, config) == pytest.approx(math.exp(log_single))


def test_parallel_member_training_matches_sequential(gpu_ok):
    """test_model.py:313-320 (`jobs` is accepted; members always train concurrently)."""
    b = _b()
    sp, ss = _training_case(n=60)
    cfg = b.TrainConfig(seed=8, epochs=30)
    seq = b.train_ensemble(ss, sp, k=3, cfg=cfg, jobs=1)
    par = b.train_ensemble(ss, sp, k=3, cfg=cfg, jobs=2)
    for x, y in zip(seq.members, par.members):
        assert np.array_equal(x.weights_hidden, y.weights_hidden)
        assert np.array_equal(x.weights_out, y.weights_out)


def test_identical_members_and_geometric_mean(gpu_ok):
    """test_model.py:330-342."""
    b = _b()
    sp = _tiny()
    enc = b.Encoder.from_space(sp)
    ens = b.Ensemble([_const_net(math.log(2.0), enc.input_dim) for _ in range(5)], enc, sp.name)
    assert b.predict(ens, sp.config_at(0)) == pytest.approx(2.0)
    ens = b.Ensemble([_const_net(0.0, enc.input_dim), _const_net(math.log(4.0), enc.input_dim)], enc, sp.name)
    assert b.predict(ens, sp.config_at(3)) == pytest.approx(2.0)


def test_predict_equals_exp_mean_of_member_logs(gpu_ok):
    """test_model.py:345-353 (rel 1e-12)."""
    b = _b()
    sp, ss = _training_case(n=80)
    ens = b.train_ensemble(ss, sp, k=4, cfg=b.TrainConfig(seed=2, epochs=60))
    for i in (0, 100, 400):
        x = ens.encoder.encode(sp.config_at(i))[np.newaxis, :]
        logs = [float(m.predict_log_batch(x)[0]) for m in ens.members]
        assert b.predict(ens, sp.config_at(i)) == pytest.approx(math.exp(sum(logs) / len(logs)), rel=1e-12)
    # and the batched device path agrees with the scalar one
    idx = np.array([0, 100, 400, 511])
    np.testing.assert_allclose(ens.predict_indices(idx), [b.predict(ens, sp.config_at(int(i))) for i in idx],
                               rtol=1e-12, atol=0)


def test_predictions_fuzz_finite_positive(gpu_ok):
    """test_model.py:356-363 (make_rng(77) = PCG64 seeded 77)."""
    b = _b()
    sp, ss = _training_case(n=150)
    ens = b.train_ensemble(ss, sp, k=3, cfg=b.TrainConfig(seed=4, epochs=80))
    idx = np.random.Generator(np.random.PCG64(77)).integers(0, sp.cardinality(), size=10_000)
    preds = ens.predict_indices(idx)
    assert np.isfinite(preds).all() and (preds > 0).all()


# ---- test_paramspace.py -------------------------------------------------------------

def test_mixed_radix_matches_itertools_enumeration(gpu_ok):
    """test_paramspace.py:72-78 on the device decode, plus the whole tiny space."""
    b = _b()
    sp = b.ParamSpace("two", (b.ParamDef("a", (1, 2, 4)), b.ParamDef("b", (0, 1))))
    assert [tuple(r) for r in sp.decode_indices(np.arange(sp.cardinality()))] == \
        list(itertools.product((1, 2, 4), (0, 1)))
    tiny = _tiny()
    assert [tuple(r) for r in tiny.decode_indices(np.arange(tiny.cardinality()))] == \
        list(itertools.product(*(p.values for p in tiny.params)))


def test_valid_count_matches_brute_force(gpu_ok):
    """test_paramspace.py:197-210 with all three rule kinds: brute force over
    itertools == scalar rule checks == the device mask."""
    b = _b()
    base = _tiny()
    rules = (b.ValidityRule("max-product", ("a", "c"), (), 80),
             b.ValidityRule("max-weighted-sum", ("a", "b", "c"), (3, 5, 1), 40),
             b.ValidityRule("forbidden-combination", ("a", "b"), (2, 1), 0))
    sp = b.ParamSpace("tiny-rules", base.params, rules)

    def ok(combo):
        a, bb, c = combo
        return a * c <= 80 and 3 * a + 5 * bb + c <= 40 and not (a == 2 and bb == 1)
    brute = sum(1 for combo in itertools.product(*(p.values for p in sp.params)) if ok(combo))
    by_scalar = sum(1 for i in range(sp.cardinality()) if sp.is_statically_valid(sp.config_at(i)))
    by_mask = int(sp.valid_mask_indices(np.arange(sp.cardinality())).astype(bool).sum())
    assert brute == by_scalar == by_mask
    assert 0 < brute < sp.cardinality()


def test_encode_injective_and_rank(gpu_ok):
    """test_model.py:47-67: encode_indices == scalar encode, distinct configs
    get distinct features, values are digit / (count - 1)."""
    b = _b()
    sp = _tiny()
    enc = b.Encoder.from_space(sp)
    feats = enc.encode_indices(np.arange(sp.cardinality()))
    for i in range(sp.cardinality()):
        assert np.array_equal(feats[i], enc.encode(sp.config_at(i)))
    assert len({tuple(r) for r in feats.tolist()}) == sp.cardinality()
    assert enc.encode((2, 1, 40)).tolist() == [0.5, 1.0, 1.0]
