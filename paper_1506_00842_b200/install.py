"""Drop-in rebinding for an installed reference package `mltune`.

    import mltune, paper_1506_00842_b200 as b200
    b200.install()            # mltune.autotune now sweeps and trains on the B200

Rebinds the module globals the reference resolves at call time:
`mltune.tuner.top_m_predicted` and `mltune.tuner.train_ensemble`
(autotune looks both up as module globals, tuner.py:25, :152, :155),
`mltune.evaluation.train_ensemble` (evaluation.py:22, :134),
`mltune.cli.train_ensemble` (cli.py:44-49, :324: `mltune train`),
`mltune.model.train_ensemble / train_network` and the package-level
re-exports (__init__.py:44-61). Native errors then raise the reference's own
exception classes. The replacements take the reference's own objects
(ParamSpace, SampleSet, TrainConfig, Ensemble) structurally — see
tests/test_dropin_reference.py, which drives the real `mltune` through here.
"""

from __future__ import annotations

import importlib

from . import errors, model, tuner

_saved: dict = {}


def install(mltune_module=None) -> None:
    mt = mltune_module or importlib.import_module("mltune")
    ref_err = importlib.import_module(mt.__name__ + ".errors")
    for name in list(errors.active):
        errors.active[name] = getattr(ref_err, name, errors.active[name])
    targets = [(mt.tuner, "top_m_predicted", tuner.top_m_predicted),
               (mt.tuner, "train_ensemble", model.train_ensemble),
               (mt.evaluation, "train_ensemble", model.train_ensemble),
               (mt, "top_m_predicted", tuner.top_m_predicted),
               (mt, "train_ensemble", model.train_ensemble)]
    for sub, names in (("model", ("train_ensemble", "train_network")), ("cli", ("train_ensemble",))):
        try:
            mod = importlib.import_module(f"{mt.__name__}.{sub}")
        except ImportError:
            continue
        targets += [(mod, n, getattr(model, n)) for n in names if hasattr(mod, n)]
    if hasattr(mt, "train_network"):
        targets.append((mt, "train_network", model.train_network))
    for mod, attr, fn in targets:
        _saved.setdefault((mod.__name__, attr), (mod, getattr(mod, attr)))
        setattr(mod, attr, fn)


def uninstall() -> None:
    for (_, attr), (mod, fn) in list(_saved.items()):
        setattr(mod, attr, fn)
    _saved.clear()
    for name in list(errors.active):
        errors.active[name] = getattr(errors, name)
