"""Performance model — the API surface of `mltune.model`
(/root/reference/pkg/src/mltune/model.py) with prediction and training on
the B200.

* `Ensemble.predict_indices / predict_features / predict` run the fp64
  device kernel (A3-A6; model.py:88-97, :146-170, :290-301).
* `train_ensemble` / `train_network` run the fp64 device trainer (A8-A10;
  model.py:194-341). The host only does what must match the reference bit
  for bit and is not arithmetic-heavy: fold assignment, target
  standardisation and every PCG64 draw (initial weights, per-epoch
  permutations) in the reference's call order.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native as N
from . import errors
from .errors import ConfigMismatchError, ParseError
from .space import make_rng

HIDDEN_UNITS = 30
DEFAULT_BAG_COUNT = 11
MODEL_SCHEMA_VERSION = 1


@dataclass(frozen=True)
class TrainConfig:
    """model.py:30-48 (the code's defaults: lr 0.03, momentum 0.9)."""
    epochs: int = 500
    learning_rate: float = 0.03
    batch_size: int = 32
    momentum: float = 0.9
    weight_init_scale: float = 1.0
    seed: int = 0

    def __post_init__(self):
        if self.epochs < 1 or self.batch_size < 1:
            raise ValueError("epochs and batch_size must be positive")
        if not self.learning_rate > 0 or not self.weight_init_scale > 0:
            raise ValueError("learning_rate and weight_init_scale must be positive")
        if not 0.0 <= self.momentum < 1.0:
            raise ValueError("momentum must lie in [0, 1)")


class Encoder:
    """feature = rank / max(count - 1, 1) per parameter (model.py:51-111)."""

    def __init__(self, params):
        self.params = [(name, tuple(int(v) for v in values)) for name, values in params]
        self._rank = [{v: i for i, v in enumerate(vals)} for _, vals in self.params]
        self._span = [max(len(vals) - 1, 1) for _, vals in self.params]

    @classmethod
    def from_space(cls, space) -> "Encoder":
        return cls([(p.name, p.values) for p in space.params])

    @property
    def input_dim(self) -> int:
        return len(self.params)

    @property
    def counts(self) -> np.ndarray:
        return np.asarray([len(v) for _, v in self.params], dtype=np.int32)

    def index_of(self, config) -> int:
        if len(config) != len(self.params):
            raise ConfigMismatchError(f"configuration has {len(config)} values, encoder expects {len(self.params)}")
        idx = 0
        for (name, vals), rank, v in zip(self.params, self._rank, config):
            if v not in rank:
                raise ConfigMismatchError(f"value {v} is not admissible for parameter {name!r}")
            idx = idx * len(vals) + rank[v]
        return idx

    def encode(self, config) -> np.ndarray:
        return self.encode_indices([self.index_of(config)])[0]

    def encode_indices(self, indices, device=None) -> np.ndarray:
        idx = np.ascontiguousarray(indices, dtype=np.int64)
        counts = np.ascontiguousarray(self.counts)
        out = np.empty((idx.shape[0], self.input_dim), dtype=np.float64)
        if idx.shape[0]:
            N.check(N.lib().mlt_encode(N.ctx(device), N.ptr(counts, N.C.c_int32), self.input_dim,
                                       N.ptr(idx, N.C.c_int64), idx.shape[0], N.ptr(out, N.C.c_double)))
        return out

    def to_json(self) -> list:
        return [{"name": n, "values": list(v), "kind": "binary" if v == (0, 1) else "rank"} for n, v in self.params]

    @classmethod
    def from_json(cls, doc) -> "Encoder":
        return cls([(p["name"], tuple(p["values"])) for p in doc])


class Network:
    """One sigmoid network (model.py:114-170): weights_hidden (H, d),
    biases_hidden (H,), weights_out (H,), bias_out, and the target transform."""

    def __init__(self, weights_hidden, biases_hidden, weights_out, bias_out, target_mean=0.0, target_std=1.0,
                 first_epoch_loss=None, final_epoch_loss=None):
        self.weights_hidden = np.asarray(weights_hidden, dtype=np.float64)
        self.biases_hidden = np.asarray(biases_hidden, dtype=np.float64)
        self.weights_out = np.asarray(weights_out, dtype=np.float64)
        self.bias_out = float(bias_out)
        self.target_mean = float(target_mean)
        self.target_std = float(target_std)
        self.first_epoch_loss = first_epoch_loss
        self.final_epoch_loss = final_epoch_loss
        hidden = self.weights_hidden.shape[0]
        if self.biases_hidden.shape[0] != hidden or self.weights_out.shape[0] != hidden:
            raise ValueError("inconsistent network weight shapes")
        for a in (self.weights_hidden, self.biases_hidden, self.weights_out):
            if not np.all(np.isfinite(a)):
                raise ValueError("network weights must be finite")

    @property
    def input_dim(self) -> int:
        return self.weights_hidden.shape[1]

    def forward_batch(self, features) -> np.ndarray:
        """Raw (standardised) output for a feature matrix, on the device."""
        x = np.asarray(features, dtype=np.float64)
        if x.shape[-1] != self.input_dim:
            raise ValueError(f"feature length {x.shape[-1]} does not match input_dim {self.input_dim}")
        return member_outputs([self], x.reshape(-1, self.input_dim))[0].reshape(x.shape[:-1])

    def forward(self, features) -> float:
        x = np.asarray(features, dtype=np.float64)
        if x.ndim != 1:
            raise ValueError("forward expects a single feature vector")
        return float(self.forward_batch(x[np.newaxis, :])[0])

    def predict_log_batch(self, features) -> np.ndarray:
        return self.forward_batch(features) * self.target_std + self.target_mean


def forward(net: Network, features) -> float:
    return net.forward(np.asarray(features, dtype=np.float64))


def _sigmoid(z):
    with np.errstate(over="ignore"):
        return 1.0 / (1.0 + np.exp(-z))


def gradient(net: Network, features, target: float) -> dict:
    """Exact single-sample gradient of (out - target)^2 (model.py:177-191).
    A 30-element host helper (a test oracle, not on the runtime path)."""
    x = np.asarray(features, dtype=np.float64)
    if x.shape != (net.input_dim,):
        raise ValueError(f"feature shape {x.shape} does not match ({net.input_dim},)")
    h = _sigmoid(net.weights_hidden @ x + net.biases_hidden)
    g = 2.0 * (float(h @ net.weights_out + net.bias_out) - target)
    dz = g * net.weights_out * h * (1.0 - h)
    return {"weights_hidden": np.outer(dz, x), "biases_hidden": dz, "weights_out": g * h,
            "bias_out": np.array(g)}


class _Bundle:
    """Minimal ensemble-shaped view used to pack raw member weights."""

    def __init__(self, members, d):
        self.members = members
        self.encoder = Encoder([(f"x{i}", (0, 1)) for i in range(d)])


def member_outputs(members, features, device=None) -> np.ndarray:
    """[k][n] raw network outputs (forward_batch of every member) on the device."""
    x = np.ascontiguousarray(features, dtype=np.float64)
    pk = N.PackedEnsemble(_Bundle(list(members), x.shape[1]))
    out = np.empty((len(members), x.shape[0]), dtype=np.float64)
    if x.shape[0]:
        N.check(N.lib().mlt_member_outputs(N.ctx(device), N.C.byref(pk.c), N.ptr(x, N.C.c_double), x.shape[0],
                                           N.ptr(out, N.C.c_double)))
    return out


class Ensemble:
    """k networks; prediction = exp(mean of member log times) (model.py:272-301)."""

    def __init__(self, members, encoder: Encoder, space_name: str):
        if not members:
            raise ValueError("an ensemble needs at least one member")
        if {m.input_dim for m in members} != {encoder.input_dim}:
            raise ValueError("member input dimensions do not match the encoder")
        self.members = tuple(members)
        self.encoder = encoder
        self.space_name = space_name

    @property
    def k(self) -> int:
        return len(self.members)

    def predict_features(self, features) -> np.ndarray:
        return predict_features(self, features)

    def predict(self, config) -> float:
        return float(predict_indices(self, [self.encoder.index_of(config)])[0])

    def predict_indices(self, indices) -> np.ndarray:
        return predict_indices(self, indices)


def predict(ensemble, config) -> float:
    return ensemble.predict(config)


def predict_indices(ensemble, indices, device=None) -> np.ndarray:
    """fp64 exp(mean member log) for configuration indices, on the device."""
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    pk = N.packed(ensemble, "ensemble")
    out = np.empty(idx.shape[0], dtype=np.float64)
    if idx.shape[0]:
        N.check(N.lib().mlt_predict_indices(N.ctx(device), N.C.byref(pk.c), N.ptr(idx, N.C.c_int64),
                                            idx.shape[0], N.ptr(out, N.C.c_double)))
    return out


def predict_features(ensemble, features, device=None) -> np.ndarray:
    x = np.ascontiguousarray(features, dtype=np.float64)
    if x.ndim != 2:
        x = x.reshape(-1, ensemble.encoder.input_dim if hasattr(ensemble, "encoder") else x.shape[-1])
    pk = N.packed(ensemble, "ensemble")
    if x.shape[1] != pk.counts.shape[0]:
        raise ValueError(f"feature length {x.shape[1]} does not match input_dim {pk.counts.shape[0]}")
    out = np.empty(x.shape[0], dtype=np.float64)
    if x.shape[0]:
        N.check(N.lib().mlt_predict_features(N.ctx(device), N.C.byref(pk.c), N.ptr(x, N.C.c_double), x.shape[0],
                                             N.ptr(out, N.C.c_double)))
    return out


# -- training ---------------------------------------------------------------------

def _valid_rows(samples, encoder: Encoder):
    """model.py:252-258: valid samples only; X via the device encoder, y = ln t."""
    valid = [s for s in samples.samples if s.outcome.is_valid]
    if not valid:
        raise errors.active["InsufficientDataError"]("no valid samples to train on")
    idx = np.asarray([encoder.index_of(s.config) for s in valid], dtype=np.int64)
    X = encoder.encode_indices(idx)
    y = np.log([s.outcome.time for s in valid])
    return X, y


def _member_draws(n: int, d: int, cfg: TrainConfig, seed_parts):
    """Every random draw of one `_fit` in the reference's order (model.py:204-218)."""
    return _member_draws_many([(n, d, cfg, seed_parts)])[0]


def _member_draws_many(specs):
    """`_member_draws` for many members: the W1 / w2 uniforms per member in
    numpy, then every member's per-epoch permutations in one native call
    (numpy's own bit generators driven from host threads, bit-identical)."""
    rngs, inits = [], []
    for n, d, cfg, seed_parts in specs:
        rng = make_rng(*seed_parts)
        w1 = rng.uniform(-0.5, 0.5, (HIDDEN_UNITS, d)) * cfg.weight_init_scale
        w2 = rng.uniform(-0.5, 0.5, HIDDEN_UNITS) * cfg.weight_init_scale
        rngs.append(rng)
        inits.append((w1, w2))
    out = []
    by_epochs = {}
    for q, (n, d, cfg, _) in enumerate(specs):
        by_epochs.setdefault(cfg.epochs, []).append(q)
    perms = [None] * len(specs)
    for epochs, qs in by_epochs.items():
        ns = np.ascontiguousarray([specs[q][0] for q in qs], dtype=np.int32)
        buf = np.empty(int(ns.sum()) * epochs, dtype=np.int32)
        gens = (N.C.c_void_p * len(qs))(*[rngs[q].bit_generator.ctypes.bit_generator.value for q in qs])
        rc = N.lib().mlt_host_permutations(gens, len(qs), N.ptr(ns, N.C.c_int32), epochs, N.ptr(buf, N.C.c_int32), 0)
        N.check(rc, "mlt_host_permutations")
        at = 0
        for q, nq in zip(qs, ns.tolist()):
            perms[q] = buf[at:at + epochs * nq].reshape(epochs, nq)
            at += epochs * nq
    for (w1, w2), pm in zip(inits, perms):
        out.append((w1, w2, pm))
    return out


def fit_members(X, y, member_rows, cfg: TrainConfig, seed_parts, device=None) -> list:
    """Train one network per entry of `member_rows` (row indices into X/y) on the device."""
    res = fit_member_batches([(X, y, member_rows, seed_parts, cfg)], device)[0]
    if isinstance(res, Exception):
        raise res
    return res


def fit_member_batches(jobs, device=None) -> list:
    """Train the members of several independent fits in ONE device launch
    (one CTA per member, all concurrent). `jobs` = [(X, y, member_rows,
    seed_parts, cfg)]; the jobs must share the optimiser settings (epochs,
    batch size, learning rate, momentum) and the input width; each job's own
    cfg drives its host draws (init scale; the seed is in seed_parts).
    Returns, per job, its list of Networks or the DivergenceError it would
    raise alone (first diverged member in member order, as model.py:239-243)."""
    d = jobs[0][0].shape[1]
    cfg = jobs[0][4]
    opt = (cfg.epochs, cfg.batch_size, cfg.learning_rate, cfg.momentum)
    xs, ts, rows_all, n_m, iw1s, iw2s, perms, meta = [], [], [], [], [], [], [], []
    draw_specs = []
    row_base = 0
    for X, y, member_rows, seed_parts, jcfg in jobs:
        if X.shape[1] != d:
            raise ValueError("batched fits must share the input width")
        if (jcfg.epochs, jcfg.batch_size, jcfg.learning_rate, jcfg.momentum) != opt:
            raise ValueError("batched fits must share the optimiser settings")
        xs.append(np.asarray(X, dtype=np.float64))
        job_meta = []
        for rows, sp in zip(member_rows, seed_parts):
            targets = y[rows]
            mean = float(targets.mean())
            std = float(targets.std())
            if std == 0.0:
                std = 1.0
            ts.append((targets - mean) / std)
            job_meta.append((mean, std))
            draw_specs.append((len(rows), d, jcfg, sp))
            rows_all.append(np.asarray(rows) + row_base)
            n_m.append(len(rows))
        meta.append(job_meta)
        row_base += X.shape[0]
    for w1, w2, pm in _member_draws_many(draw_specs):
        iw1s.append(w1)
        iw2s.append(w2)
        perms.append(pm.ravel())
    k = len(n_m)
    x = np.ascontiguousarray(np.concatenate(xs))
    t = np.ascontiguousarray(np.concatenate(ts))
    rows = np.ascontiguousarray(np.concatenate(rows_all).astype(np.int32))
    n_m = np.asarray(n_m, dtype=np.int32)
    iw1 = np.ascontiguousarray(np.stack(iw1s))
    iw2 = np.ascontiguousarray(np.stack(iw2s))
    pall = np.ascontiguousarray(np.concatenate(perms))
    desc = N.MltTrainDesc(k, d, HIDDEN_UNITS, cfg.epochs, cfg.batch_size, cfg.learning_rate, cfg.momentum,
                          x.shape[0], N.ptr(x, N.C.c_double), N.ptr(t, N.C.c_double), N.ptr(rows, N.C.c_int32),
                          N.ptr(n_m, N.C.c_int32), N.ptr(iw1, N.C.c_double), N.ptr(iw2, N.C.c_double),
                          N.ptr(pall, N.C.c_int32))
    ow1 = np.empty((k, HIDDEN_UNITS, d))
    ob1 = np.empty((k, HIDDEN_UNITS))
    ow2 = np.empty((k, HIDDEN_UNITS))
    ob2 = np.empty(k)
    lf = np.empty(k)
    ll = np.empty(k)
    div = np.zeros(k, dtype=np.int32)
    rc = N.lib().mlt_train_members(N.ctx(device), N.C.byref(desc), N.ptr(ow1, N.C.c_double),
                                   N.ptr(ob1, N.C.c_double), N.ptr(ow2, N.C.c_double), N.ptr(ob2, N.C.c_double),
                                   N.ptr(lf, N.C.c_double), N.ptr(ll, N.C.c_double), N.ptr(div, N.C.c_int32))
    if rc != N.MLT_EDIVERGED:
        N.check(rc, "mlt_train_members")
    out, i = [], 0
    for job_meta in meta:
        dj = div[i:i + len(job_meta)]
        if dj.any():
            out.append(errors.active["DivergenceError"]("training loss became non-finite",
                                                        epoch=int(dj[np.nonzero(dj)[0][0]])))
        else:
            out.append([Network(ow1[i + q], ob1[i + q], ow2[i + q], ob2[i + q], mean, std, float(lf[i + q]),
                                float(ll[i + q])) for q, (mean, std) in enumerate(job_meta)])
        i += len(job_meta)
    return out


def train_network(samples, space, cfg: TrainConfig) -> Network:
    """A single network on all valid samples, seeded like member 0 of k=1 (model.py:261-269)."""
    enc = Encoder.from_space(space)
    X, y = _valid_rows(samples, enc)
    return fit_members(X, y, [np.arange(X.shape[0])], cfg, [(cfg.seed, 0)])[0]


def _ensemble_job(samples, space, k: int, cfg: TrainConfig):
    """Everything train_ensemble computes on the host before the device fit:
    (encoder, X, y, member rows, member seed parts) (model.py:308-341)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    enc = Encoder.from_space(space)
    X, y = _valid_rows(samples, enc)
    n = X.shape[0]
    if n < k:
        raise errors.active["InsufficientDataError"](f"{n} valid samples cannot fill {k} folds")
    if k == 1:
        rows = [np.arange(n)]
    else:
        folds = np.array_split(make_rng(cfg.seed).permutation(n), k)
        rows = [np.setdiff1d(np.arange(n), f, assume_unique=True) for f in folds]
    return enc, X, y, rows, [(cfg.seed, i) for i in range(k)]


def train_ensemble(samples, space, k: int = DEFAULT_BAG_COUNT, cfg: TrainConfig = TrainConfig(),
                   jobs: int = 1) -> Ensemble:
    """Fold-exclusion bagging (model.py:308-341); all k members train
    concurrently on the device (`jobs` is accepted for API compatibility)."""
    enc, X, y, rows, parts = _ensemble_job(samples, space, k, cfg)
    return Ensemble(fit_members(X, y, rows, cfg, parts), enc, space.name)


def train_ensembles(requests, device=None) -> list:
    """Many independent `train_ensemble(samples, space, k, cfg)` calls with
    their members trained together: one device launch per distinct
    (optimiser settings, input width). Returns, aligned with `requests`, an
    Ensemble or the exception that call would have raised. Each result is
    bit-identical to its own train_ensemble call (members are independent CTAs)."""
    out = [None] * len(requests)
    groups = {}
    for q, (samples, space, k, cfg) in enumerate(requests):
        try:
            enc, X, y, rows, parts = _ensemble_job(samples, space, k, cfg)
        except Exception as exc:   # ValueError / InsufficientDataError (ours or, install()ed, the reference's)
            out[q] = exc
            continue
        key = (cfg.epochs, cfg.batch_size, cfg.learning_rate, cfg.momentum, X.shape[1])
        groups.setdefault(key, []).append((q, enc, space.name, (X, y, rows, parts, cfg)))
    for items in groups.values():
        res = fit_member_batches([it[3] for it in items], device)
        for (q, enc, name, _), r in zip(items, res):
            out[q] = r if isinstance(r, Exception) else Ensemble(r, enc, name)
    return out


# -- persistence (schema v1, model.py:351-410) ----------------------------------------

def _fmt(obj) -> str:
    """JSON with floats to 17 significant digits (serialize.py:9-27)."""
    if isinstance(obj, float):
        if not math.isfinite(obj):
            raise ValueError("cannot serialize non-finite float")
        return format(obj, ".17g")
    if isinstance(obj, bool) or obj is None or isinstance(obj, (int, str)):
        return json.dumps(obj)
    if isinstance(obj, (list, tuple)):
        return "[" + ", ".join(_fmt(v) for v in obj) + "]"
    if isinstance(obj, dict):
        return "{" + ", ".join(f"{json.dumps(k)}: {_fmt(v)}" for k, v in obj.items()) + "}"
    raise TypeError(f"cannot serialize {type(obj).__name__}")


def model_to_json(ens) -> dict:
    return {"schema_version": MODEL_SCHEMA_VERSION, "space_name": ens.space_name, "k": len(ens.members),
            "input_dim": ens.encoder.input_dim, "encoder": ens.encoder.to_json(),
            "target_transform": [{"mean": m.target_mean, "std": m.target_std} for m in ens.members],
            "members": [{"weights_hidden": m.weights_hidden.tolist(), "biases_hidden": m.biases_hidden.tolist(),
                         "weights_out": m.weights_out.tolist(), "bias_out": m.bias_out} for m in ens.members]}


def save_model(ens, path) -> None:
    Path(path).write_text(_fmt(model_to_json(ens)) + "\n")


def model_from_json(doc: dict, path="<json>") -> Ensemble:
    try:
        if doc["schema_version"] != MODEL_SCHEMA_VERSION:
            raise ParseError(f"unsupported model schema version {doc['schema_version']}", path=path)
        enc = Encoder.from_json(doc["encoder"])
        members = [Network(np.asarray(m["weights_hidden"], dtype=np.float64),
                           np.asarray(m["biases_hidden"], dtype=np.float64),
                           np.asarray(m["weights_out"], dtype=np.float64), float(m["bias_out"]),
                           float(t["mean"]), float(t["std"]))
                   for m, t in zip(doc["members"], doc["target_transform"], strict=True)]
        if len(members) != doc["k"]:
            raise ParseError("member count does not match k", path=path)
        if doc["input_dim"] != enc.input_dim:
            raise ParseError("input_dim does not match encoder", path=path)
        return Ensemble(members, enc, doc["space_name"])
    except ParseError:
        raise
    except (KeyError, TypeError, ValueError) as exc:
        raise ParseError(f"bad model file: {exc}", path=path) from exc


def load_model(path) -> Ensemble:
    path = Path(path)
    try:
        doc = json.loads(path.read_text())
    except json.JSONDecodeError as exc:
        raise ParseError(f"not a valid model file: {exc}", path=path) from exc
    return model_from_json(doc, path)
