"""§8(f) next #4: the batched evaluation harness against the reference's own
learning_curve / slowdown_grid / random_baseline on the 512-configuration
test space (tests/golden/eval_bench512.json, make_golden.py --eval). The
runner is the reference-pinned oracle surrogate, so only the device training
and sweep differ from the reference run."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN, oracle_space, product_space

pytestmark = pytest.mark.gpu


class _OracleRunner:
    """SurrogateRunner semantics over the oracle (bit-exact with the reference)."""

    default_repetitions = 1

    def __init__(self, doc, space_name, runner_id="s512"):
        from oracle.surrogate import OSurrogate
        self.s = OSurrogate(doc, oracle_space(space_name))
        self.sp = product_space(space_name)
        self.runner_id = runner_id

    def measure(self, config, repetitions=None):
        import paper_1506_00842_b200 as b
        reps = repetitions or 1
        t, ok = self.s.measured_times(np.array([self.sp.index_of(config)]), reps)
        return b.Sample(tuple(config), b.Outcome.valid(float(t[0])) if ok[0] else b.Outcome.invalid("invalid-launch"),
                        reps)

    def measured_times(self, idx, reps=1):
        return self.s.measured_times(np.asarray(idx), reps)


@pytest.fixture(scope="module")
def fixture():
    return json.loads((GOLDEN / "eval_bench512.json").read_text())


def test_learning_curve_matches_reference(gpu_ok, fixture):
    from paper_1506_00842_b200 import evaluation as EV
    sizes, repeats, seed, k, hold = fixture["args"]["learning_curve"]
    pts = EV.learning_curve(product_space("bench512"), _OracleRunner(fixture["surrogate"], "bench512"), sizes,
                            repeats, seed, k=k, holdout_size=hold)
    for p, want in zip(pts, fixture["learning_curve"]):
        assert p.n_train == want["n_train"] and list(p.failure_reasons) == want["failure_reasons"]
        np.testing.assert_allclose(p.repeat_mres, want["repeat_mres"], rtol=1e-9)
        assert p.mre == pytest.approx(want["mre"], rel=1e-9)


def test_slowdown_grid_matches_reference(gpu_ok, fixture, tmp_path):
    from paper_1506_00842_b200 import evaluation as EV
    nv, mv, repeats, seed, k = fixture["args"]["slowdown_grid"]
    cells = EV.slowdown_grid(product_space("bench512"), _OracleRunner(fixture["surrogate"], "bench512"), nv, mv,
                             repeats, seed, k=k)
    for c, want in zip(cells, fixture["slowdown_grid"]):
        assert (c.n_train, c.m_candidates, c.n_repeats, c.invalid_run_count) == \
            (want["n_train"], want["m_candidates"], want["n_repeats"], want["invalid_run_count"])
        assert c.mean_slowdown == pytest.approx(want["mean_slowdown"], rel=1e-12)
    out = tmp_path / "grid.csv"
    EV.write_slowdown_grid_csv(cells, out)
    assert out.read_text().splitlines()[0] == "n_train,m_candidates,mean_slowdown,n_success,n_invalid"


def test_slowdown_grid_on_the_device_surrogate(gpu_ok, fixture):
    """The same grid with the device surrogate as the runner (exhaustive optimum
    from the fused kernel; noisy times within 1e-13 of the reference)."""
    from paper_1506_00842_b200 import B200SurrogateRunner
    from paper_1506_00842_b200 import evaluation as EV
    nv, mv, repeats, seed, k = fixture["args"]["slowdown_grid"]
    r = B200SurrogateRunner(fixture["surrogate"], product_space("bench512"), runner_id="s512")
    cells = EV.slowdown_grid(product_space("bench512"), r, nv, mv, repeats, seed, k=k)
    for c, want in zip(cells, fixture["slowdown_grid"]):
        assert c.mean_slowdown == pytest.approx(want["mean_slowdown"], rel=1e-9)


def test_random_baseline_and_batched_training_identity(gpu_ok, fixture):
    """random_baseline matches; train_ensembles == train_ensemble one by one, bit for bit."""
    import paper_1506_00842_b200 as b
    from paper_1506_00842_b200 import evaluation as EV
    from paper_1506_00842_b200.model import train_ensembles
    sp = product_space("bench512")
    run = _OracleRunner(fixture["surrogate"], "bench512")
    n, seed = fixture["args"]["random_baseline"]
    cfg, t = EV.random_baseline(sp, run, n, seed)
    assert list(cfg) == fixture["random_baseline"]["config"] and t == fixture["random_baseline"]["time"]
    sets = [b.SampleSet(sp, "s", tuple(b.measure_configs(sp, run, sp.sample_random(60 + 20 * i, i)))) for i in range(4)]
    reqs = [(ss, sp, 3, b.TrainConfig(seed=i, epochs=40)) for i, ss in enumerate(sets)]
    reqs.append((b.SampleSet(sp, "s", ()), sp, 3, b.TrainConfig(epochs=40)))      # no valid samples
    many = train_ensembles(reqs)
    assert isinstance(many[-1], b.InsufficientDataError)
    for (ss, _, k, cfg), e in zip(reqs[:-1], many[:-1]):
        one = b.train_ensemble(ss, sp, k=k, cfg=cfg)
        for m1, m2 in zip(one.members, e.members):
            assert np.array_equal(m1.weights_hidden, m2.weights_hidden) and m1.bias_out == m2.bias_out
