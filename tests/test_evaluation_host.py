"""The evaluation harness's host orchestration (seeds, sampling streams,
holdout exclusion, run ordering, failure bookkeeping, cell aggregation) on
CPU: the device trainer / sweep / predictor are swapped for the oracle (the
reference's own arithmetic), so learning_curve and slowdown_grid must
reproduce the reference's outputs on the 512-configuration test space
EXACTLY (tests/golden/eval_bench512.json, written by make_golden.py --eval)."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN, oracle_space, product_space


class _OracleRunner:
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


class _OracleEnsemble:
    """What train_ensembles returns, backed by the oracle (reference arithmetic)."""

    def __init__(self, oens, osp, psp):
        self.oens, self.osp, self.psp = oens, osp, psp
        outer = self

        class _Enc:
            def encode(self, config):
                return outer.osp.encode(np.array([outer.psp.index_of(config)]))[0]

        self.encoder = _Enc()


@pytest.fixture
def oracle_device(monkeypatch):
    """Route the harness's device calls to the oracle."""
    import paper_1506_00842_b200 as b
    from oracle.model import OEnsemble, OTrainCfg, fit, fold_rows
    from oracle.tuner import top_m
    from paper_1506_00842_b200 import evaluation as EV
    from paper_1506_00842_b200 import tuner as T

    def train_ensembles(requests, device=None):
        out = []
        for samples, space, k, cfg in requests:
            osp = oracle_space(space.name)
            valid = [s for s in samples.samples if s.outcome.is_valid]
            if len(valid) < max(k, 1):
                out.append(b.InsufficientDataError("not enough valid samples"))
                continue
            idx = np.array([space.index_of(s.config) for s in valid], dtype=np.int64)
            X = osp.encode(idx)
            y = np.log([s.outcome.time for s in valid])
            ocfg = OTrainCfg(epochs=cfg.epochs, learning_rate=cfg.learning_rate, batch_size=cfg.batch_size,
                             momentum=cfg.momentum, weight_init_scale=cfg.weight_init_scale, seed=cfg.seed)
            rows = fold_rows(X.shape[0], k, cfg.seed)
            nets = [fit(X[r], y[r], ocfg, (cfg.seed, i)) for i, r in enumerate(rows)]
            out.append(_OracleEnsemble(OEnsemble(nets, osp.radix), osp, space))
        return out

    def predict_features(ens, feats, device=None):
        return ens.oens.predict_features(np.asarray(feats))

    def top_m_predicted(ens, space, m, sweep_cap=None, seed=0):
        i, p = top_m(ens.oens, ens.osp, m, sweep_cap, seed)
        return [(space.config_at(int(q)), float(v)) for q, v in zip(i, p)]

    monkeypatch.setattr(EV, "train_ensembles", train_ensembles)
    monkeypatch.setattr(EV, "predict_features", predict_features)
    monkeypatch.setattr(T, "top_m_predicted", top_m_predicted)


@pytest.fixture(scope="module")
def fixture():
    return json.loads((GOLDEN / "eval_bench512.json").read_text())


def test_learning_curve_host_logic_exact(oracle_device, fixture):
    from paper_1506_00842_b200 import evaluation as EV
    sizes, repeats, seed, k, hold = fixture["args"]["learning_curve"]
    pts = EV.learning_curve(product_space("bench512"), _OracleRunner(fixture["surrogate"], "bench512"), sizes,
                            repeats, seed, k=k, holdout_size=hold)
    got = [{"n_train": p.n_train, "mre": p.mre, "repeat_mres": list(p.repeat_mres),
            "failure_reasons": list(p.failure_reasons)} for p in pts]
    assert got == fixture["learning_curve"]


def test_slowdown_grid_host_logic_exact(oracle_device, fixture, tmp_path):
    from paper_1506_00842_b200 import evaluation as EV
    nv, mv, repeats, seed, k = fixture["args"]["slowdown_grid"]
    cells = EV.slowdown_grid(product_space("bench512"), _OracleRunner(fixture["surrogate"], "bench512"), nv, mv,
                             repeats, seed, k=k)
    got = [{"n_train": c.n_train, "m_candidates": c.m_candidates, "mean_slowdown": c.mean_slowdown,
            "n_repeats": c.n_repeats, "invalid_run_count": c.invalid_run_count} for c in cells]
    assert got == fixture["slowdown_grid"]
    EV.write_slowdown_grid_csv(cells, tmp_path / "g.csv")
    rows = (tmp_path / "g.csv").read_text().splitlines()
    assert rows[0] == "n_train,m_candidates,mean_slowdown,n_success,n_invalid" and len(rows) == len(cells) + 1


def test_random_baseline_host_exact(fixture, monkeypatch):
    from paper_1506_00842_b200 import evaluation as EV
    n, seed = fixture["args"]["random_baseline"]
    sp = product_space("bench512")

    r = _OracleRunner(fixture["surrogate"], "bench512")
    osp = oracle_space("bench512")                    # host stand-ins for the device decode / mask
    monkeypatch.setattr(type(sp), "decode_indices", lambda self, idx: osp.decode(np.asarray(idx)))
    monkeypatch.setattr(type(sp), "static_valid_mask", lambda self, vm: osp.rule_mask(osp.rules, vm))
    cfg, t = EV.random_baseline(sp, r, n, seed)
    assert list(cfg) == fixture["random_baseline"]["config"] and t == fixture["random_baseline"]["time"]
