"""Oracle: the analytic surrogate device (`mltune/measurement.py:114-238`).

Used by tests to produce stage-1 samples and exhaustive ground truth on the
GPU box, where the reference package is absent. Test infrastructure only.
"""

from __future__ import annotations

import numpy as np
from scipy.special import ndtri

from .space import ORule

_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)


def _mix(x):
    """measurement.py:125-132 — splitmix64 finalizer."""
    x = x.astype(np.uint64, copy=True)
    x ^= x >> np.uint64(30)
    x *= _C1
    x ^= x >> np.uint64(27)
    x *= _C2
    x ^= x >> np.uint64(31)
    return x


def normals(seed: int, idx, rep: int):
    """measurement.py:135-142."""
    i = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _mix(np.uint64(seed & ((1 << 64) - 1)) + _G * (i + np.uint64(1)))
        h = _mix(h + _G * np.uint64((rep + 1) & ((1 << 32) - 1)))
    return ndtri(((h >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -53)


class OSurrogate:
    """measurement.py:193-258 over a spec JSON (measurement.py:497-554 schema)."""

    def __init__(self, doc: dict, space, runner_id="surrogate", default_repetitions=1):
        pos = {n: i for i, n in enumerate(space.names)}
        self.space = space
        self.base = float(doc["base_time"])
        self.terms = [([pos[p] for p in t["params"]], [int(v) for v in t["match"]],
                       float(t["factor"])) for t in doc.get("terms", ())]
        self.cv = float(doc.get("noise_cv", 0.0))
        self.seed = int(doc.get("seed", 0))
        self.rules = []
        for r in doc.get("invalid_rules", ()):
            co = tuple(int(c) for c in r.get("coefficients", ()))
            if not co and r["kind"] != "forbidden-combination":
                co = (1,) * len(r["operands"])
            self.rules.append(ORule(r["kind"], tuple(pos[o] for o in r["operands"]),
                                    co, int(r.get("bound", 0))))
        self.runner_id = runner_id
        self.default_repetitions = default_repetitions

    def true_times(self, idx):
        vm = self.space.decode(idx)
        ok = self.space.rule_mask(self.rules, vm)
        t = np.full(vm.shape[0], self.base)
        for ps, ms, f in self.terms:
            hit = np.ones(vm.shape[0], dtype=bool)
            for p, v in zip(ps, ms):
                hit &= vm[:, p] == v
            t[hit] *= f
        t[~ok] = np.nan
        return t, ok

    def measured_times(self, idx, reps: int = 1):
        t, ok = self.true_times(idx)
        if self.cv > 0:
            z = normals(self.seed, idx, 0)
            for r in range(1, reps):
                z = np.minimum(z, normals(self.seed, idx, r))
            t = t * np.exp(float(np.sqrt(np.log1p(self.cv ** 2))) * z)
        return t, ok
