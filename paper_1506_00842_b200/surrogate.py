"""The analytic surrogate device on the B200 — `mltune.measurement`'s
SurrogateRunner (/root/reference/pkg/src/mltune/measurement.py:146-258)
evaluated by `k_surr_times`, plus a fused exhaustive search
(`k_surr_best`, tuner.py:191-224) that sweeps a whole space on the device.

Noise-free times are bit-identical to the reference (same factor product
order); noisy times use CUDA's normcdfinv/exp in place of scipy's ndtri and
glibc's exp and agree to ~1e-15 relative. Specs are the reference's
SurrogateSpec objects or their JSON form (measurement.py:497-554).
"""

from __future__ import annotations

import math

import numpy as np

from . import _native as N
from . import errors
from .measurement import STATUS_INVALID_LAUNCH, Outcome, Sample


def _get(spec, name, default=None):
    if isinstance(spec, dict):
        return spec.get(name, default)
    return getattr(spec, name, default)


class PackedSurrogate:
    """mlt_surrogate over host arrays kept alive by this object."""

    def __init__(self, spec, space):
        pos = {p.name: i for i, p in enumerate(space.params)}
        terms = list(_get(spec, "terms", ()) or ())
        T = len(terms)
        self.nparams = np.zeros(max(T, 1), dtype=np.int32)
        self.tpos = np.zeros((max(T, 1), 2), dtype=np.int32)
        self.match = np.zeros((max(T, 1), 2), dtype=np.int64)
        self.factor = np.ones(max(T, 1), dtype=np.float64)
        for t, term in enumerate(terms):
            ps = list(_get(term, "params"))
            ms = [int(v) for v in _get(term, "match")]
            if len(ps) not in (1, 2) or len(ps) != len(ms):
                raise ValueError("surrogate terms cover one parameter or a pair")
            self.nparams[t] = len(ps)
            for j, (p, v) in enumerate(zip(ps, ms)):
                if p not in pos:
                    raise errors.active["ConfigMismatchError"](f"surrogate term names unknown parameter {p!r}")
                self.tpos[t, j] = pos[p]
                self.match[t, j] = v
            self.factor[t] = float(_get(term, "factor"))
        rules = list(_get(spec, "invalid_rules", ()) or ())
        for r in rules:
            for o in (r["operands"] if isinstance(r, dict) else r.operands):
                if o not in pos:
                    raise errors.active["ConfigMismatchError"](f"surrogate rule names unknown parameter {o!r}")
        self.kind, self.nops, self.rpos, self.coeff, self.bound = N.pack_rules(rules, pos)
        cv = float(_get(spec, "noise_cv", 0.0) or 0.0)
        # SurrogateSpec.log_sigma (measurement.py:187-190), computed with numpy exactly as there
        self.log_sigma = float(np.sqrt(np.log1p(cv ** 2)))
        self.noise = cv > 0
        self.base_time = float(_get(spec, "base_time"))
        if not self.base_time > 0:
            raise ValueError("base_time must be strictly positive")
        self.seed = int(_get(spec, "seed", 0) or 0) & ((1 << 64) - 1)
        self.c = N.MltSurrogate(self.base_time, T, N.ptr(self.nparams, N.C.c_int32), N.ptr(self.tpos, N.C.c_int32),
                                N.ptr(self.match, N.C.c_int64), N.ptr(self.factor, N.C.c_double),
                                self.log_sigma if self.noise else 0.0, self.seed, len(rules),
                                N.ptr(self.kind, N.C.c_int32), N.ptr(self.nops, N.C.c_int32),
                                N.ptr(self.rpos, N.C.c_int32), N.ptr(self.coeff, N.C.c_int64),
                                N.ptr(self.bound, N.C.c_int64))


class B200SurrogateRunner:
    """Deterministic synthetic device evaluated on the GPU; the interface of
    the reference SurrogateRunner (measurement.py:193-258)."""

    def __init__(self, spec, space, runner_id: str = "surrogate", default_repetitions: int = 1, device=None):
        self.spec = spec
        self.space = space
        self.runner_id = runner_id
        self.default_repetitions = default_repetitions
        self.device = device
        self._pk = PackedSurrogate(spec, space)

    def _times(self, indices, reps):
        idx = np.ascontiguousarray(indices, dtype=np.int64).reshape(-1)
        times = np.empty(idx.shape[0], dtype=np.float64)
        ok = np.empty(idx.shape[0], dtype=np.uint8)
        if idx.shape[0]:
            ps = N.packed(self.space, "space")
            rc = N.lib().mlt_surrogate_times(N.ctx(self.device), N.C.byref(ps.c), N.C.byref(self._pk.c),
                                             N.ptr(idx, N.C.c_int64), idx.shape[0], int(reps),
                                             N.ptr(times, N.C.c_double), N.ptr(ok, N.C.c_uint8))
            N.check(rc, "mlt_surrogate_times")
        return times, ok.astype(bool)

    def true_times(self, indices):
        """Noise-free times; NaN where a launch rule fires (measurement.py:212-226)."""
        return self._times(indices, 0)

    def measured_times(self, indices, repetitions: int = 1):
        """Noisy times, min over repetitions (measurement.py:228-238)."""
        if repetitions < 1:
            raise ValueError("repetitions must be >= 1")
        return self._times(indices, repetitions)

    def true_time(self, config) -> float:
        times, ok = self.true_times([self.space.index_of(config)])
        if not ok[0]:
            raise errors.active["InvalidConfigurationError"](
                f"configuration {config} violates a launch rule of the surrogate")
        return float(times[0])

    def measure(self, config, repetitions: int | None = None) -> Sample:
        reps = self.default_repetitions if repetitions is None else repetitions
        if reps < 1:
            raise ValueError("repetitions must be >= 1")
        times, ok = self.measured_times([self.space.index_of(config)], reps)
        if not ok[0]:
            return Sample(tuple(config), Outcome.invalid(STATUS_INVALID_LAUNCH), reps)
        return Sample(tuple(config), Outcome.valid(float(times[0])), reps)

    def measure_many(self, configs, repetitions: int | None = None) -> list:
        """`measure` of many configurations in one device call (same results)."""
        reps = self.default_repetitions if repetitions is None else repetitions
        if reps < 1:
            raise ValueError("repetitions must be >= 1")
        configs = [tuple(c) for c in configs]
        if not configs:
            return []
        idx = np.fromiter((self.space.index_of(c) for c in configs), dtype=np.int64, count=len(configs))
        times, ok = self.measured_times(idx, reps)
        return [Sample(c, Outcome.valid(float(t)) if good else Outcome.invalid(STATUS_INVALID_LAUNCH), reps)
                for c, t, good in zip(configs, times.tolist(), ok.tolist())]

    def exhaustive_best(self, begin: int = 0, end: int | None = None, repetitions: int | None = None,
                        threshold: float = math.nan):
        """Device exhaustive search over [begin, end): (best index or -1, best
        time, valid count, count strictly faster than `threshold`)."""
        reps = self.default_repetitions if repetitions is None else int(repetitions)
        ps = N.packed(self.space, "space")
        end = ps.card if end is None else int(end)
        bi, bt, nv, nb = N.C.c_int64(), N.C.c_double(), N.C.c_int64(), N.C.c_int64()
        rc = N.lib().mlt_surrogate_best(N.ctx(self.device), N.C.byref(ps.c), N.C.byref(self._pk.c), int(begin), end,
                                        reps, float(threshold), N.C.byref(bi), N.C.byref(bt), N.C.byref(nv),
                                        N.C.byref(nb))
        N.check(rc, "mlt_surrogate_best")
        return int(bi.value), float(bt.value), int(nv.value), int(nb.value)
