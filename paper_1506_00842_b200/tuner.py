"""Two-stage auto-tuning — the API of `mltune.tuner`
(/root/reference/pkg/src/mltune/tuner.py) with the full-space sweep on the B200.

`top_m_predicted` is the drop-in for tuner.py:95-131. It never materialises
the space: the device decodes every index, evaluates the ensemble in fp32
with an a-priori error bound, keeps every configuration within the guard
band of the running m-th best, rescores those in fp64 in the reference's
operation order and sorts by (prediction, index) — the reference's
`lexsort((indices, preds))`. The orchestration around it (`autotune`,
`measure_configs`, `exhaustive_search`) is host logic over duck-typed runners,
as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import errors
from .measurement import STATUS_INVALID_STATIC, Outcome, Sample, SampleSet
from .model import DEFAULT_BAG_COUNT, TrainConfig, train_ensemble

SWEEP_CHUNK = 1 << 17
REPORT_SCHEMA_VERSION = 1


@dataclass(frozen=True)
class TunerConfig:
    """tuner.py:33-53."""
    n_train: int
    m_candidates: int
    k_bag: int = DEFAULT_BAG_COUNT
    seed: int = 0
    train_cfg: TrainConfig | None = None
    max_prediction_sweep: int | None = None

    def __post_init__(self):
        if self.m_candidates < 1:
            raise ValueError("m_candidates must be >= 1")
        if self.n_train < self.k_bag:
            raise ValueError("n_train must be at least k_bag")
        if self.max_prediction_sweep is not None and self.max_prediction_sweep < 1:
            raise ValueError("max_prediction_sweep must be >= 1 when set")

    def resolved_train_cfg(self) -> TrainConfig:
        return self.train_cfg if self.train_cfg is not None else TrainConfig(seed=self.seed)


@dataclass(frozen=True)
class TuningReport:
    """tuner.py:56-77."""
    space_name: str
    runner_id: str
    config: TunerConfig
    stage1_samples: SampleSet
    stage2_samples: SampleSet
    stage2_invalid_count: int
    best_config: tuple | None = None
    best_index: int | None = None
    best_time: float | None = None
    predicted_best_time: float | None = None

    @property
    def measurements_total(self) -> int:
        return len(self.stage1_samples) + len(self.stage2_samples)


MLT_OPT_PRUNE = N.MLT_OPT_PRUNE


def set_sweep_pruning(on: bool, device=None) -> None:
    """Exact bound-based pruning in the device sweep (mlt_ctx_set_option
    MLT_OPT_PRUNE): a work item stops once every configuration in it provably
    exceeds the running threshold. Results are identical either way; off by
    default, so every configuration of the space is evaluated."""
    N.check(N.lib().mlt_ctx_set_option(N.ctx(device), MLT_OPT_PRUNE, 1 if on else 0), "mlt_ctx_set_option")


def top_m_arrays(ensemble, space, m: int, begin: int = 0, end: int | None = None, indices=None,
                 device=None, with_stats: bool = False):
    """Device top-m over the slice [begin, end) of `space` (or over an index
    list) -> (indices int64, predictions float64[, stats dict])."""
    if m < 1:
        raise ValueError("m must be >= 1")
    ps = N.packed(space, "space")
    pe = N.packed(ensemble, "ensemble")
    card = ps.card
    end = card if end is None else int(end)
    out_idx = np.empty(m, dtype=np.int64)
    out_pred = np.empty(m, dtype=np.float64)
    out_n = N.C.c_int64(0)
    st = N.MltSweepStats()
    if indices is not None:
        lst = np.ascontiguousarray(indices, dtype=np.int64)
        rc = N.lib().mlt_top_m(N.ctx(device), N.C.byref(ps.c), N.C.byref(pe.c), int(m), int(begin), end,
                               N.ptr(lst, N.C.c_int64), lst.shape[0], N.ptr(out_idx, N.C.c_int64),
                               N.ptr(out_pred, N.C.c_double), N.C.byref(out_n), N.C.byref(st))
        N.check(rc, "mlt_top_m")
    else:
        # slices run on the resident plan of (space, ensemble): descriptors and
        # factored tables persist across calls with the same objects
        plan = N.plan(space, ensemble, device)
        rc = N.lib().mlt_plan_top_m(plan.h, int(m), int(begin), end, N.ptr(out_idx, N.C.c_int64),
                                    N.ptr(out_pred, N.C.c_double), N.C.byref(out_n), N.C.byref(st))
        N.check(rc, "mlt_plan_top_m")
    n = out_n.value
    res = (out_idx[:n].copy(), out_pred[:n].copy())
    return res + (st.as_dict(),) if with_stats else res


def configs_of(space, indices) -> list:
    """Configuration tuples of `indices`. Works on any space object the
    reference's `top_m_predicted` accepts: this package's ParamSpace has a
    batched `configs_at`; the reference's has only the scalar `config_at`
    (paramspace.py:149-158), which is what its own sweep uses (tuner.py:131)."""
    batched = getattr(space, "configs_at", None)
    if batched is not None:
        return batched(indices)
    return [space.config_at(int(i)) for i in indices]


def top_m_predicted(ensemble, space, m: int, sweep_cap: int | None = None, seed: int = 0) -> list:
    """The m statically-valid configurations with the lowest predicted times,
    ascending, ties broken by index; fewer when fewer are valid (tuner.py:95-131)."""
    if m < 1:
        raise ValueError("m must be >= 1")
    card = space.cardinality()
    if sweep_cap is not None and card > sweep_cap:
        subset = np.sort(space.sample_indices(sweep_cap, seed))   # host RNG: the reference stream
        idx, pred = top_m_arrays(ensemble, space, m, indices=subset)
    else:
        idx, pred = top_m_arrays(ensemble, space, m)
    return list(zip(configs_of(space, idx), pred.tolist()))


def measure_configs(space, runner, configs, repetitions: int | None = None) -> list:
    """Static invalids never reach the runner (tuner.py:80-92). A runner with
    `measure_many(configs, repetitions)` (the device surrogate) measures the
    statically valid ones in one batch; otherwise one `measure` per config."""
    reps_default = repetitions if repetitions is not None else getattr(runner, "default_repetitions", 1)
    out = [None] * len(configs)
    todo = []
    for q, config in enumerate(configs):
        if space.is_statically_valid(config):
            todo.append(q)
        else:
            out[q] = Sample(config, Outcome.invalid(STATUS_INVALID_STATIC), reps_default)
    if hasattr(runner, "measure_many"):
        for q, smp in zip(todo, runner.measure_many([configs[q] for q in todo], repetitions)):
            out[q] = smp
    else:
        for q in todo:
            out[q] = runner.measure(configs[q], repetitions)
    return out


def autotune(space, runner, cfg: TunerConfig, jobs: int = 1, sweep=None) -> TuningReport:
    """Sample -> measure -> train (device) -> sweep + top-M (device) -> re-measure
    -> best of stage 2 by (time, index) (tuner.py:134-188). `sweep` may replace
    the top-M function (e.g. the multi-GPU `distributed.top_m_predicted`)."""
    stage1 = autotune_stage1(space, runner, cfg)
    ens = train_ensemble(stage1, space, k=cfg.k_bag, cfg=cfg.resolved_train_cfg(), jobs=jobs)
    return autotune_stage2(space, runner, cfg, stage1, ens, sweep)


def autotune_stage1(space, runner, cfg: TunerConfig) -> SampleSet:
    """The first half of autotune up to training: the seeded sample, measured,
    with the valid-count check (tuner.py:145-151)."""
    if space.cardinality() < cfg.n_train:
        raise ValueError(f"n_train={cfg.n_train} exceeds space cardinality {space.cardinality()}")
    rid = getattr(runner, "runner_id", "runner")
    stage1 = SampleSet(space, rid, tuple(measure_configs(space, runner, space.sample_random(cfg.n_train, cfg.seed))))
    n_valid = len(stage1.valid_samples())
    if n_valid < cfg.k_bag:
        raise errors.active["InsufficientDataError"](
            f"stage 1 produced {n_valid} valid samples, need at least {cfg.k_bag}")
    return stage1


def autotune_stage2(space, runner, cfg: TunerConfig, stage1, ens, sweep=None) -> TuningReport:
    """The second half of autotune after training (tuner.py:155-188): device
    sweep + top-M, re-measure, best by (time, index)."""
    rid = getattr(runner, "runner_id", "runner")
    sweep = sweep or top_m_predicted
    cands = sweep(ens, space, cfg.m_candidates, cfg.max_prediction_sweep, cfg.seed)
    predicted = {space.index_of(c): p for c, p in cands}
    stage2 = SampleSet(space, rid, tuple(measure_configs(space, runner, [c for c, _ in cands])))
    best, invalid = None, 0
    for s in stage2.samples:
        if not s.outcome.is_valid:
            invalid += 1
            continue
        key = (s.outcome.time, space.index_of(s.config))
        if best is None or key < best:
            best = key
    if best is None:
        partial = TuningReport(space.name, rid, cfg, stage1, stage2, invalid)
        raise errors.active["AllCandidatesInvalidError"](
            f"all {len(stage2)} second-stage candidates were invalid", report=partial)
    t, i = best
    return TuningReport(space.name, rid, cfg, stage1, stage2, invalid, best_config=space.config_at(i),
                        best_index=i, best_time=t, predicted_best_time=predicted[i])


def exhaustive_search(space, runner):
    """Measure every statically valid configuration once; return the fastest
    (tuner.py:191-224). Vectorised through `runner.measured_times` when present."""
    card = space.cardinality()
    best = None
    if hasattr(runner, "exhaustive_best"):      # device surrogate: one fused sweep of the whole space
        i, t, n_valid, _ = runner.exhaustive_best()
        if n_valid > 0:
            best = (t, i)
    elif hasattr(runner, "measured_times"):
        reps = getattr(runner, "default_repetitions", 1)
        for s in range(0, card, SWEEP_CHUNK):
            idx = np.arange(s, min(s + SWEEP_CHUNK, card), dtype=np.int64)
            if getattr(space, "rules", ()):
                idx = idx[space.valid_mask_indices(idx)] if hasattr(space, "valid_mask_indices") else \
                    idx[space.static_valid_mask(space.decode_indices(idx))]
            if idx.size == 0:
                continue
            times, ok = runner.measured_times(idx, reps)
            if not ok.any():
                continue
            pos = int(np.nanargmin(np.where(ok, times, np.nan)))
            key = (float(times[pos]), int(idx[pos]))
            if best is None or key < best:
                best = key
    else:
        for i in range(card):
            c = space.config_at(i)
            if not space.is_statically_valid(c):
                continue
            smp = runner.measure(c)
            if smp.outcome.is_valid and (best is None or (smp.outcome.time, i) < best):
                best = (smp.outcome.time, i)
    if best is None:
        raise errors.active["EmptySpaceError"](f"space {space.name!r} has no valid configuration")
    return space.config_at(best[1]), best[0]
