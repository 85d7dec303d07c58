"""On-disk formats of the tuner, read and written by
this package so the reference's CLI files interoperate with the device path:

* sample CSV (mltune.measurement.SampleWriter / save_samples / load_samples /
  measured_indices, /root/reference/pkg/src/mltune/measurement.py:353-494):
  a `# mltune-samples space=<name> runner=<id>` line, a header
  `config_index,<params...>,status,time_seconds,repetitions`, one row per
  sample, times as 17 significant digits, invalid rows with an empty time;
* surrogate spec JSON (measurement.py:497-554) with the SurrogateTerm /
  SurrogateSpec records;
* the prediction CSV of `mltune predict` (cli.py:330-353,
  `config_index,predicted_seconds`), produced here from device predictions
  in large chunks with native multi-threaded formatting (the reference
  formats one row per Python call, its next host bottleneck after the sweep).

Model JSON lives in model.py (save_model / load_model).
"""

from __future__ import annotations

import csv
import json
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native as N
from . import errors
from .measurement import ALL_STATUSES, STATUS_VALID, Outcome, Sample, SampleSet
from .space import BUILTIN_SPACE_NAMES, ValidityRule, builtin_space

SAMPLES_MAGIC = "# mltune-samples"
PRED_HEADER = "config_index,predicted_seconds\n"


def _parse_error(msg, path=None, line=None):
    return errors.active["ParseError"](msg, path=path, line=line)


def fmt17(t: float) -> str:
    """17 significant digits: every double round-trips exactly."""
    return format(float(t), ".17g")


def _columns(space) -> list:
    return ["config_index"] + list(space.param_names()) + ["status", "time_seconds", "repetitions"]


# ---- sample CSV ------------------------------------------------------------------

class SampleWriter:
    """Row-at-a-time sample CSV writer, flushed per row so an interrupted
    measurement campaign keeps what it measured (measurement.py:360-394);
    `append=True` continues a non-empty file without a second header."""

    def __init__(self, path, space, runner_id: str, append: bool = False):
        self.path = Path(path)
        self.space = space
        cont = append and self.path.exists() and self.path.stat().st_size > 0
        self._fh = open(self.path, "a" if cont else "w", newline="")
        self._csv = csv.writer(self._fh, lineterminator="\n")
        if not cont:
            self._fh.write(f"{SAMPLES_MAGIC} space={space.name} runner={runner_id}\n")
            self._csv.writerow(_columns(space))
            self._fh.flush()

    def write(self, sample) -> None:
        o = sample.outcome
        self._csv.writerow([self.space.index_of(sample.config), *sample.config, o.status,
                            fmt17(o.time) if o.is_valid else "", sample.repetitions])
        self._fh.flush()

    def close(self) -> None:
        self._fh.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def save_samples(sample_set, path) -> None:
    with SampleWriter(path, sample_set.space, sample_set.runner_id) as w:
        for s in sample_set.samples:
            w.write(s)


def load_samples(path, space=None) -> SampleSet:
    """Parse a sample CSV; the space comes from the metadata line when it
    names a built-in space, else it must be passed (and must match)."""
    path = Path(path)
    with open(path, newline="") as fh:
        first = fh.readline().rstrip("\n")
        if not first.startswith(SAMPLES_MAGIC):
            raise _parse_error("missing sample-set metadata line", path, 1)
        meta = {}
        for tok in first[len(SAMPLES_MAGIC):].split():
            if "=" in tok:
                k, v = tok.split("=", 1)
                meta[k] = v
        sname, runner_id = meta.get("space", ""), meta.get("runner", "unknown")
        if space is None:
            if sname not in BUILTIN_SPACE_NAMES:
                raise _parse_error(f"space {sname!r} is not built in; pass the space explicitly", path, 1)
            space = builtin_space(sname)
        elif space.name != sname:
            raise _parse_error(f"file holds samples for space {sname!r}, not {space.name!r}", path, 1)
        rows = csv.reader(fh)
        header = next(rows, None)
        if header is None:
            raise _parse_error("missing header row", path, 2)
        want = _columns(space)
        if header != want:
            raise _parse_error(f"header {header} does not match expected {want}", path, 2)
        P = len(space.params)
        out = []
        for ln, row in enumerate(rows, start=3):
            if not row:
                continue
            if len(row) != len(want):
                raise _parse_error(f"expected {len(want)} fields, got {len(row)}", path, ln)
            try:
                index = int(row[0])
                config = tuple(int(v) for v in row[1:1 + P])
                status, ttext, reps = row[1 + P], row[2 + P], int(row[3 + P])
            except ValueError as exc:
                raise _parse_error(str(exc), path, ln) from exc
            try:
                space.validate_config(config)
            except Exception as exc:
                raise _parse_error(str(exc), path, ln) from exc
            if space.index_of(config) != index:
                raise _parse_error(f"config_index {index} does not match configuration {config}", path, ln)
            if status not in ALL_STATUSES:
                raise _parse_error(f"unknown status {status!r}", path, ln)
            if status == STATUS_VALID:
                try:
                    outcome = Outcome.valid(float(ttext))
                except ValueError as exc:
                    raise _parse_error(str(exc), path, ln) from exc
            else:
                if ttext:
                    raise _parse_error("invalid rows must have an empty time_seconds", path, ln)
                outcome = Outcome.invalid(status)
            out.append(Sample(config, outcome, reps))
    return SampleSet(space=space, runner_id=runner_id, samples=tuple(out))


def measured_indices(path, space=None) -> set:
    """Indices already in a sample CSV (resume support, measurement.py:488-494)."""
    ss = load_samples(path, space)
    return {ss.space.index_of(s.config) for s in ss.samples}


# ---- surrogate spec JSON -----------------------------------------------------------

@dataclass(frozen=True)
class SurrogateTerm:
    """Multiplicative effect when every named parameter takes its matched value
    (measurement.py:148-166)."""
    params: tuple
    match: tuple
    factor: float

    def __post_init__(self):
        object.__setattr__(self, "params", tuple(self.params))
        object.__setattr__(self, "match", tuple(int(v) for v in self.match))
        if len(self.params) not in (1, 2):
            raise ValueError("surrogate terms cover one parameter or a pair")
        if len(self.params) != len(self.match):
            raise ValueError("term params and match values differ in length")
        if not self.factor > 0:
            raise ValueError("term factors must be strictly positive")


@dataclass(frozen=True)
class SurrogateSpec:
    """Analytic device model (measurement.py:168-190)."""
    base_time: float
    terms: tuple = ()
    noise_cv: float = 0.0
    invalid_rules: tuple = ()
    seed: int = 0

    def __post_init__(self):
        object.__setattr__(self, "terms", tuple(self.terms))
        object.__setattr__(self, "invalid_rules", tuple(self.invalid_rules))
        if not self.base_time > 0:
            raise ValueError("base_time must be strictly positive")
        if self.noise_cv < 0:
            raise ValueError("noise_cv must be non-negative")

    @property
    def log_sigma(self) -> float:
        return float(np.sqrt(np.log1p(self.noise_cv ** 2)))


def surrogate_to_json(spec) -> dict:
    return {"base_time": spec.base_time,
            "terms": [{"params": list(t.params), "match": list(t.match), "factor": t.factor} for t in spec.terms],
            "noise_cv": spec.noise_cv,
            "invalid_rules": [{"kind": r.kind, "operands": list(r.operands), "coefficients": list(r.coefficients),
                               "bound": r.bound} for r in spec.invalid_rules],
            "seed": spec.seed}


def surrogate_from_json(doc: dict, source="<json>") -> SurrogateSpec:
    try:
        return SurrogateSpec(
            base_time=float(doc["base_time"]),
            terms=tuple(SurrogateTerm(tuple(t["params"]), tuple(t["match"]), float(t["factor"]))
                        for t in doc.get("terms", ())),
            noise_cv=float(doc.get("noise_cv", 0.0)),
            invalid_rules=tuple(ValidityRule(r["kind"], tuple(r["operands"]), tuple(r.get("coefficients", ())),
                                             int(r.get("bound", 0))) for r in doc.get("invalid_rules", ())),
            seed=int(doc.get("seed", 0)))
    except (KeyError, TypeError, ValueError) as exc:
        raise _parse_error(f"bad surrogate spec: {exc}", source) from exc


def save_surrogate_spec(spec, path) -> None:
    Path(path).write_text(json.dumps(surrogate_to_json(spec), indent=2) + "\n")


def load_surrogate_spec(path) -> SurrogateSpec:
    path = Path(path)
    try:
        doc = json.loads(path.read_text())
    except json.JSONDecodeError as exc:
        raise _parse_error(f"not valid JSON: {exc}", path) from exc
    return surrogate_from_json(doc, source=path)


# ---- prediction CSV (mltune predict) -------------------------------------------------

def format_prediction_rows(indices, preds) -> str:
    """`index,prediction` lines with the prediction as '.17g' (cli.py:346-351),
    formatted natively on host threads (mlt_format_predictions)."""
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    p = np.ascontiguousarray(preds, dtype=np.float64)
    if idx.shape != p.shape:
        raise ValueError("indices and predictions differ in length")
    n = idx.shape[0]
    if n == 0:
        return ""
    cap = n * 48
    buf = N.C.create_string_buffer(cap)
    used = N.C.c_int64(0)
    N.check(N.lib().mlt_format_predictions(N.ptr(idx, N.C.c_int64), N.ptr(p, N.C.c_double), n, buf, cap,
                                           N.C.byref(used), 0), "mlt_format_predictions")
    return buf.raw[:used.value].decode("ascii")


def write_predictions_csv(ensemble, path, indices=None, chunk: int = 1 << 20, device=None) -> int:
    """The file `mltune predict --model M --out F [--index I]` writes: every
    configuration of the model's space (or the given indices), predicted on
    the device in chunks of `chunk`. Returns the row count."""
    from .model import predict_indices
    card = math.prod(len(vals) for _, vals in ensemble.encoder.params)
    idx_all = np.arange(card, dtype=np.int64) if indices is None else np.asarray(indices, dtype=np.int64)
    if idx_all.size and (idx_all.min() < 0 or idx_all.max() >= card):
        raise ValueError(f"index out of range for {card} configurations")
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    with open(path, "w", newline="") as fh:
        fh.write(PRED_HEADER)
        for s in range(0, idx_all.shape[0], chunk):
            part = idx_all[s:s + chunk]
            fh.write(format_prediction_rows(part, predict_indices(ensemble, part, device=device)))
    return int(idx_all.shape[0])
