"""Oracle: sigmoid-MLP ensemble forward pass and mini-batch SGD training.

Restates `mltune/model.py` (paths relative to /root/reference/pkg/src/mltune).
Test infrastructure only — see oracle/__init__.py. The arithmetic is written
with the same numpy/BLAS calls in the same order as the reference so the
oracle reproduces it bit-for-bit on the same numpy build.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .space import make_rng

HIDDEN = 30                                   # model.py:25


@dataclass
class ONet:
    W1: np.ndarray     # (H, d)
    b1: np.ndarray     # (H,)
    w2: np.ndarray     # (H,)
    b2: float
    mean: float = 0.0
    std: float = 1.0
    first_loss: float = math.nan
    final_loss: float = math.nan


def sigmoid(z):
    """model.py:167-170."""
    with np.errstate(over="ignore"):
        return 1.0 / (1.0 + np.exp(-z))


def net_out(net: ONet, X: np.ndarray) -> np.ndarray:
    """model.py:146-154 — raw (standardized) output."""
    h = sigmoid(np.asarray(X, dtype=np.float64) @ net.W1.T + net.b1)
    return h @ net.w2 + net.b2


def net_log(net: ONet, X) -> np.ndarray:
    """model.py:162-164 — de-standardized log time (two roundings, no FMA)."""
    return net_out(net, X) * net.std + net.mean


class OEnsemble:
    """model.py:272-301 — geometric mean over members (mean in log space)."""

    def __init__(self, nets, counts):
        self.nets = list(nets)
        self.counts = list(counts)          # encoder value counts per feature

    def mean_log(self, X) -> np.ndarray:
        logs = net_log(self.nets[0], X)
        for n in self.nets[1:]:
            logs = logs + net_log(n, X)
        return logs / len(self.nets)

    def predict_features(self, X) -> np.ndarray:     # model.py:290-294
        return np.exp(self.mean_log(X))

    def encode(self, idx) -> np.ndarray:             # model.py:88-97
        rem = np.asarray(idx, dtype=np.int64).copy()
        out = np.empty((rem.shape[0], len(self.counts)), dtype=np.float64)
        for col in reversed(range(len(self.counts))):
            rem, dig = np.divmod(rem, self.counts[col])
            out[:, col] = dig / max(self.counts[col] - 1, 1)
        return out

    def predict_indices(self, idx) -> np.ndarray:    # model.py:300-301
        return self.predict_features(self.encode(idx))


def ensemble_from_doc(doc: dict) -> OEnsemble:
    """Model JSON schema v1 (model.py:351-410)."""
    nets = []
    for m, t in zip(doc["members"], doc["target_transform"]):
        nets.append(ONet(np.asarray(m["weights_hidden"], dtype=np.float64),
                         np.asarray(m["biases_hidden"], dtype=np.float64),
                         np.asarray(m["weights_out"], dtype=np.float64),
                         float(m["bias_out"]), float(t["mean"]), float(t["std"])))
    return OEnsemble(nets, [len(p["values"]) for p in doc["encoder"]])


@dataclass
class OTrainCfg:
    """model.py:30-48 defaults (the code's values, not the SPEC's)."""
    epochs: int = 500
    learning_rate: float = 0.03
    batch_size: int = 32
    momentum: float = 0.9
    weight_init_scale: float = 1.0
    seed: int = 0


class ODivergence(Exception):
    def __init__(self, epoch):
        super().__init__(f"training loss became non-finite at epoch {epoch}")
        self.epoch = epoch


def fit(X, y, cfg: OTrainCfg, seed_parts) -> ONet:
    """model.py:194-249 — standardize, U(-1/2,1/2) init in RNG order W1 then
    w2, per-epoch permutation, momentum SGD on mean squared error."""
    n, d = X.shape
    mean = float(y.mean())
    std = float(y.std())
    if std == 0.0:
        std = 1.0
    t = (y - mean) / std
    rng = make_rng(*seed_parts)
    W1 = rng.uniform(-0.5, 0.5, (HIDDEN, d)) * cfg.weight_init_scale
    b1 = np.zeros(HIDDEN)
    w2 = rng.uniform(-0.5, 0.5, HIDDEN) * cfg.weight_init_scale
    b2 = 0.0
    vW1, vb1, vw2, vb2 = np.zeros_like(W1), np.zeros_like(b1), np.zeros_like(w2), 0.0
    lr, mu = cfg.learning_rate, cfg.momentum
    first = last = math.nan
    for epoch in range(1, cfg.epochs + 1):
        perm = rng.permutation(n)
        sse = 0.0
        for s in range(0, n, cfg.batch_size):
            rows = perm[s:s + cfg.batch_size]
            Xb, tb, m = X[rows], t[rows], rows.size
            h = sigmoid(Xb @ W1.T + b1)
            r = (h @ w2 + b2) - tb
            sse += float(r @ r)
            g = (2.0 / m) * r
            dz = np.outer(g, w2) * h * (1.0 - h)
            vW1 = mu * vW1 - lr * (dz.T @ Xb)
            vb1 = mu * vb1 - lr * dz.sum(axis=0)
            vw2 = mu * vw2 - lr * (h.T @ g)
            vb2 = mu * vb2 - lr * g.sum()
            W1 += vW1
            b1 += vb1
            w2 += vw2
            b2 += vb2
        loss = sse / n
        if not math.isfinite(loss):
            raise ODivergence(epoch)
        if epoch == 1:
            first = loss
        last = loss
    return ONet(W1, b1, w2, b2, mean, std, first, last)


def fold_rows(n: int, k: int, seed: int):
    """model.py:326-333 — fold-exclusion bagging: member i keeps every row
    outside fold i of a seeded permutation split into k near-equal folds."""
    if k == 1:
        return [np.arange(n)]
    folds = np.array_split(make_rng(seed).permutation(n), k)
    return [np.setdiff1d(np.arange(n), f, assume_unique=True) for f in folds]


def train(X, y, k: int, cfg: OTrainCfg) -> list:
    """model.py:308-341 (sequential; jobs>1 is bit-identical by construction)."""
    return [fit(X[rows], y[rows], cfg, (cfg.seed, i))
            for i, rows in enumerate(fold_rows(X.shape[0], k, cfg.seed))]
