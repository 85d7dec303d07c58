"""The drop-in boundary driven by the REAL reference package.

`paper_1506_00842_b200.install()` rebinds the module globals of an imported
`mltune` (tuner.py:25, :152, :155; evaluation.py:22, :134). These tests import
the unmodified reference — `baseline/_ref` (its pip install, which travels to
the GPU box) or `/root/reference/pkg/src` (build container) — install the B200
path into it and run the reference's OWN `autotune`, `learning_curve` and
`slowdown_grid` on the reference's own ParamSpace / SurrogateRunner / Ensemble
objects, comparing with the reference's recorded outputs
(tests/golden/eval_bench512.json, make_golden.py --eval) and with the
un-installed reference on the same inputs.

* CPU tests (`-m "not gpu"`): the device calls of this package are replaced by
  the oracle (test infrastructure), so they check the glue — attribute access
  on reference objects, exception classes, result shapes — not the kernels.
* GPU tests: the same calls with the real device path (libmltune_b200.so).
"""

from __future__ import annotations

import importlib
import json
import math
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, golden, model_doc, spaces_doc

_REF_DIRS = [ROOT / "baseline" / "_ref", ROOT.parent / "reference" / "pkg" / "src"]


def _import_reference():
    for d in _REF_DIRS:
        if (d / "mltune" / "__init__.py").exists():
            if str(d) not in sys.path:
                sys.path.insert(0, str(d))
            mt = importlib.import_module("mltune")
            importlib.import_module("mltune.cli")
            return mt
    return None


@pytest.fixture(scope="module")
def mt():
    mod = _import_reference()
    if mod is None:
        pytest.skip("the reference package is not importable here (no baseline/_ref, no /root/reference)")
    return mod


@pytest.fixture(scope="module")
def evalfix():
    return json.loads((GOLDEN / "eval_bench512.json").read_text())


def _ref_space(mt, name):
    return mt.paramspace.space_from_json(spaces_doc()[name])


def _ref_runner(mt, evalfix, space):
    spec = mt.measurement.surrogate_from_json(evalfix["surrogate"])
    return mt.SurrogateRunner(spec, space, runner_id="s512")


@pytest.fixture
def installed(mt):
    import paper_1506_00842_b200 as b200
    b200.install(mt)
    try:
        yield mt
    finally:
        b200.uninstall()


# ---- oracle stand-ins for the device calls (CPU tests only) --------------------------

@pytest.fixture
def oracle_device(monkeypatch):
    """Replace every device call the drop-in path makes with the oracle, so the
    host glue can be checked without a GPU."""
    from oracle.model import OEnsemble, ONet, ODivergence, OTrainCfg, fit
    from oracle.tuner import top_m as o_top_m
    from paper_1506_00842_b200 import errors, model, tuner

    def o_ens(ens):
        nets = [ONet(np.asarray(m.weights_hidden), np.asarray(m.biases_hidden), np.asarray(m.weights_out),
                     float(m.bias_out), float(m.target_mean), float(m.target_std)) for m in ens.members]
        return OEnsemble(nets, [len(v) for _, v in ens.encoder.params])

    def fit_member_batches(jobs, device=None):
        out = []
        for X, y, member_rows, seed_parts, cfg in jobs:
            ocfg = OTrainCfg(cfg.epochs, cfg.learning_rate, cfg.batch_size, cfg.momentum, cfg.weight_init_scale,
                             cfg.seed)
            try:
                nets = [fit(X[rows], y[rows], ocfg, sp) for rows, sp in zip(member_rows, seed_parts)]
            except ODivergence as e:
                out.append(errors.active["DivergenceError"]("training loss became non-finite", epoch=e.epoch))
                continue
            out.append([model.Network(n.W1, n.b1, n.w2, n.b2, n.mean, n.std, n.first_loss, n.final_loss)
                        for n in nets])
        return out

    class _OSpace:
        def __init__(self, space):
            from oracle.space import space_from_doc
            pk = space
            doc = {"name": getattr(pk, "name", "s"),
                   "params": [{"name": p.name, "values": list(p.values)} for p in pk.params],
                   "rules": [{"kind": r.kind, "operands": list(r.operands), "coefficients": list(r.coefficients),
                              "bound": r.bound} for r in getattr(pk, "rules", ())]}
            self.o = space_from_doc(doc)

    def top_m_arrays(ensemble, space, m, begin=0, end=None, indices=None, device=None, with_stats=False):
        osp = _OSpace(space).o
        if indices is not None:
            idx = np.asarray(indices, dtype=np.int64)
            idx = idx[osp.valid_mask(osp.decode(idx))]
            pred = o_ens(ensemble).predict_indices(idx)
            order = np.lexsort((idx, pred))[:m]
            res = (idx[order], pred[order])
        else:
            res = o_top_m(o_ens(ensemble), osp, m, begin=begin, end=end)
        return res + ({},) if with_stats else res

    def encode_indices(self, indices, device=None):
        rem = np.asarray(indices, dtype=np.int64).copy()
        out = np.empty((rem.shape[0], len(self.params)), dtype=np.float64)
        for col in reversed(range(len(self.params))):
            c = len(self.params[col][1])
            rem, dig = np.divmod(rem, c)
            out[:, col] = dig / max(c - 1, 1)
        return out

    monkeypatch.setattr(model, "fit_member_batches", fit_member_batches)
    monkeypatch.setattr(model.Encoder, "encode_indices", encode_indices)
    monkeypatch.setattr(model, "predict_features", lambda ens, x, device=None: o_ens(ens).predict_features(
        np.asarray(x, dtype=np.float64).reshape(-1, ens.encoder.input_dim)))
    monkeypatch.setattr(model, "predict_indices", lambda ens, i, device=None: o_ens(ens).predict_indices(
        np.asarray(i, dtype=np.int64)))
    monkeypatch.setattr(tuner, "top_m_arrays", top_m_arrays)
    return True


# ---- the checks (shared by the CPU and GPU variants) ----------------------------------

def _check_autotune_equals_reference(mt, evalfix):
    """The reference's own autotune, B200 path installed, vs the reference alone."""
    import paper_1506_00842_b200 as b200
    sp = _ref_space(mt, "bench512")
    cfg = mt.TunerConfig(n_train=120, m_candidates=16, k_bag=3, seed=11)
    got = mt.autotune(sp, _ref_runner(mt, evalfix, sp), cfg)
    assert isinstance(got, mt.TuningReport)
    b200.uninstall()
    want = mt.autotune(sp, _ref_runner(mt, evalfix, sp), cfg)
    b200.install(mt)
    assert got.best_index == want.best_index and got.best_config == want.best_config
    assert got.best_time == want.best_time
    assert math.isclose(got.predicted_best_time, want.predicted_best_time, rel_tol=1e-9)
    assert [s.config for s in got.stage2_samples.samples] == [s.config for s in want.stage2_samples.samples]


def _check_learning_curve(mt, evalfix):
    sizes, repeats, seed, k, hold = evalfix["args"]["learning_curve"]
    sp = _ref_space(mt, "bench512")
    pts = mt.learning_curve(sp, _ref_runner(mt, evalfix, sp), sizes, repeats, seed, k=k, holdout_size=hold)
    for p, want in zip(pts, evalfix["learning_curve"]):
        assert p.n_train == want["n_train"] and list(p.failure_reasons) == want["failure_reasons"]
        np.testing.assert_allclose(p.repeat_mres, want["repeat_mres"], rtol=1e-9)


def _check_slowdown_grid(mt, evalfix):
    nv, mv, repeats, seed, k = evalfix["args"]["slowdown_grid"]
    sp = _ref_space(mt, "bench512")
    cells = mt.slowdown_grid(sp, _ref_runner(mt, evalfix, sp), nv, mv, repeats, seed, k=k)
    for c, want in zip(cells, evalfix["slowdown_grid"]):
        assert (c.n_train, c.m_candidates, c.invalid_run_count) == (want["n_train"], want["m_candidates"],
                                                                    want["invalid_run_count"])
        assert c.mean_slowdown == pytest.approx(want["mean_slowdown"], rel=1e-12)


def _check_top_m_on_reference_objects(mt, tmp_path):
    """top_m_predicted on a reference Ensemble (mltune.load_model) over a
    reference ParamSpace: the golden top-m of that model."""
    p = tmp_path / "conv_k11.json"
    p.write_text(json.dumps(model_doc("conv_k11")))
    ens = mt.load_model(p)
    sp = mt.builtin_space("convolution") if "convolution" in mt.BUILTIN_SPACE_NAMES else \
        _ref_space(mt, "convolution")
    res = mt.top_m_predicted(ens, sp, 10)
    g = golden("topm_conv_k11.npz")
    assert [sp.index_of(c) for c, _ in res] == g["m10_i"].tolist()
    np.testing.assert_allclose([t for _, t in res], g["m10_p"], rtol=1e-12)
    assert all(isinstance(c, tuple) for c, _ in res)
    with pytest.raises(ValueError):
        mt.top_m_predicted(ens, sp, 0)


def _check_errors_are_reference_classes(mt, evalfix):
    sp = _ref_space(mt, "bench512")
    runner = _ref_runner(mt, evalfix, sp)
    ss = mt.SampleSet(sp, "s512", tuple(mt.tuner.measure_configs(sp, runner, sp.sample_random(2, 0))))
    with pytest.raises(mt.InsufficientDataError):
        mt.tuner.train_ensemble(ss, sp, k=5)


# ---- CPU (oracle stand-ins) -----------------------------------------------------------

def test_install_rebinds_every_reference_entry(installed):
    import paper_1506_00842_b200 as b200
    mt = installed
    assert mt.tuner.top_m_predicted is b200.top_m_predicted
    assert mt.tuner.train_ensemble is b200.train_ensemble
    assert mt.evaluation.train_ensemble is b200.train_ensemble
    assert mt.cli.train_ensemble is b200.train_ensemble
    assert mt.model.train_network is b200.model.train_network


def test_uninstall_restores_the_reference(mt):
    import paper_1506_00842_b200 as b200
    orig = (mt.tuner.top_m_predicted, mt.tuner.train_ensemble, mt.evaluation.train_ensemble, mt.cli.train_ensemble)
    b200.install(mt)
    b200.uninstall()
    assert (mt.tuner.top_m_predicted, mt.tuner.train_ensemble, mt.evaluation.train_ensemble,
            mt.cli.train_ensemble) == orig


def test_glue_autotune(installed, oracle_device, evalfix):
    _check_autotune_equals_reference(installed, evalfix)


def test_glue_learning_curve(installed, oracle_device, evalfix):
    _check_learning_curve(installed, evalfix)


def test_glue_slowdown_grid(installed, oracle_device, evalfix):
    _check_slowdown_grid(installed, evalfix)


def test_glue_top_m_on_reference_objects(installed, oracle_device, tmp_path):
    _check_top_m_on_reference_objects(installed, tmp_path)


def test_glue_errors(installed, oracle_device, evalfix):
    _check_errors_are_reference_classes(installed, evalfix)


def test_packing_reference_objects_equals_product_objects(mt, tmp_path):
    """The C descriptors built from reference objects are the ones built from
    this package's objects (no device needed: packing is host-only)."""
    from conftest import product_ensemble, product_space
    from paper_1506_00842_b200 import _native as N
    p = tmp_path / "m.json"
    p.write_text(json.dumps(model_doc("conv_k11")))
    a, b = N.PackedEnsemble(mt.load_model(p)), N.PackedEnsemble(product_ensemble("conv_k11"))
    for f in ("counts", "w1", "b1", "w2", "b2", "mean", "std"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    for name in ("conv-rules", "bench512", "synthetic-1e8"):
        a, b = N.PackedSpace(_ref_space(mt, name)), N.PackedSpace(product_space(name))
        for f in ("radix", "values", "kind", "nops", "rpos", "coeff", "bound"):
            np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
        assert a.card == b.card


# ---- GPU (the real device path) ------------------------------------------------------

@pytest.mark.gpu
def test_gpu_dropin_autotune(gpu_ok, installed, evalfix):
    _check_autotune_equals_reference(installed, evalfix)


@pytest.mark.gpu
def test_gpu_dropin_learning_curve(gpu_ok, installed, evalfix):
    _check_learning_curve(installed, evalfix)


@pytest.mark.gpu
def test_gpu_dropin_slowdown_grid(gpu_ok, installed, evalfix):
    _check_slowdown_grid(installed, evalfix)


@pytest.mark.gpu
def test_gpu_dropin_top_m_on_reference_objects(gpu_ok, installed, tmp_path):
    _check_top_m_on_reference_objects(installed, tmp_path)


@pytest.mark.gpu
def test_gpu_dropin_errors(gpu_ok, installed, evalfix):
    _check_errors_are_reference_classes(installed, evalfix)


@pytest.mark.gpu
def test_gpu_integration_snippet_verbatim(gpu_ok, mt):
    """INTEGRATION.md §1, as written there (smaller budgets)."""
    import paper_1506_00842_b200 as b200
    space = mt.builtin_space("convolution")
    runner = mt.SurrogateRunner(mt.builtin_surrogate("gpu-a", space), space)
    b200.install()
    try:
        report = mt.autotune(space, runner, mt.TunerConfig(n_train=300, m_candidates=20))
    finally:
        b200.uninstall()
    want = mt.autotune(space, runner, mt.TunerConfig(n_train=300, m_candidates=20))
    assert report.best_index == want.best_index and report.best_time == want.best_time
