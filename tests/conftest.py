"""Shared test plumbing: the `gpu` marker, golden-fixture loaders, and the
oracle (tests are one of the few places allowed to import oracle/)."""

from __future__ import annotations

import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libmltune_b200.so")


@lru_cache(maxsize=None)
def spaces_doc() -> dict:
    return json.loads((GOLDEN / "spaces.json").read_text())


@lru_cache(maxsize=None)
def surrogates_doc() -> dict:
    return json.loads((GOLDEN / "surrogates.json").read_text())


def product_space(name):
    from paper_1506_00842_b200.space import space_from_json
    return space_from_json(spaces_doc()[name])


def oracle_space(name):
    from oracle.space import space_from_doc
    return space_from_doc(spaces_doc()[name])


@lru_cache(maxsize=None)
def model_doc(case) -> dict:
    return json.loads((GOLDEN / f"model_{case}.json").read_text())


def product_ensemble(case):
    from paper_1506_00842_b200.model import model_from_json
    return model_from_json(model_doc(case))


def oracle_ensemble(case):
    from oracle.model import ensemble_from_doc
    return ensemble_from_doc(model_doc(case))


def golden(name) -> dict:
    with np.load(GOLDEN / name) as z:
        return {k: z[k] for k in z.files}


CASE_SPACE = {"conv_k1": "convolution", "conv_k11": "convolution", "raycast_k11": "raycasting",
              "stereo_k8": "stereo", "synth_k16": "synthetic-1e8", "b512_k3": "bench512"}


@pytest.fixture(scope="session")
def gpu_ok():
    from paper_1506_00842_b200 import _native as N
    N.ctx(0)   # raises NativeUnavailableError without a B200: the GPU tests must not pass silently
    return True


def oracle_of_product_ensemble(ens):
    """The oracle restatement of an in-memory product (or reference) Ensemble."""
    from oracle.model import OEnsemble, ONet
    nets = [ONet(np.asarray(m.weights_hidden, dtype=np.float64), np.asarray(m.biases_hidden, dtype=np.float64),
                 np.asarray(m.weights_out, dtype=np.float64), float(m.bias_out), float(m.target_mean),
                 float(m.target_std)) for m in ens.members]
    return OEnsemble(nets, [len(v) for _, v in ens.encoder.params])


def oracle_of_product_space(sp):
    """The oracle restatement of an in-memory ParamSpace (product or reference)."""
    from oracle.space import space_from_doc
    return space_from_doc({"name": sp.name,
                           "params": [{"name": p.name, "values": list(p.values)} for p in sp.params],
                           "rules": [{"kind": r.kind, "operands": list(r.operands),
                                      "coefficients": list(r.coefficients), "bound": int(r.bound)}
                                     for r in getattr(sp, "rules", ())]})
