"""Oracle: configuration-space indexing, validity rules and sampling.

Restates `mltune/paramspace.py` (reference paths relative to
/root/reference/pkg/src/mltune). Test infrastructure only — see
oracle/__init__.py.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

PERMUTATION_LIMIT = 1 << 22          # paramspace.py:35


def make_rng(*parts: int) -> np.random.Generator:
    """rng.py:15-22 — PCG64 seeded from a SeedSequence of 64-bit-wrapped parts."""
    return np.random.default_rng(
        np.random.SeedSequence([int(p) & ((1 << 64) - 1) for p in parts]))


@dataclass
class ORule:
    """paramspace.py:53-107 — kind in {max-product, max-weighted-sum,
    forbidden-combination}; positions are parameter indices."""
    kind: str
    positions: tuple
    coeffs: tuple
    bound: int


class OSpace:
    """Mixed-radix space, last parameter fastest (paramspace.py:110-193)."""

    def __init__(self, name, names, values, rules=()):
        self.name = name
        self.names = list(names)
        self.values = [tuple(int(v) for v in vs) for vs in values]
        self.radix = [len(v) for v in self.values]
        self.rules = list(rules)

    @property
    def card(self) -> int:                       # paramspace.py:137-138
        return math.prod(self.radix)

    def decode(self, idx) -> np.ndarray:
        """paramspace.py:184-193: (n,) int64 -> (n, P) value matrix."""
        rem = np.asarray(idx, dtype=np.int64).copy()
        out = np.empty((rem.shape[0], len(self.radix)), dtype=np.int64)
        for col in reversed(range(len(self.radix))):
            rem, dig = np.divmod(rem, self.radix[col])
            out[:, col] = np.asarray(self.values[col], dtype=np.int64)[dig]
        return out

    def config_at(self, index: int) -> tuple:    # paramspace.py:149-158
        return tuple(int(v) for v in self.decode(np.array([index]))[0])

    def index_of(self, config) -> int:           # paramspace.py:160-166
        idx = 0
        for vals, v in zip(self.values, config):
            idx = idx * len(vals) + vals.index(int(v))
        return idx

    def rule_mask(self, rules, vm: np.ndarray) -> np.ndarray:
        """paramspace.py:92-107 + 205-213. int64 arithmetic wraps like numpy."""
        ok = np.ones(vm.shape[0], dtype=bool)
        with np.errstate(over="ignore"):
            for r in rules:
                cols = [vm[:, p] for p in r.positions]
                if r.kind == "max-product":
                    acc = np.ones(vm.shape[0], dtype=np.int64)
                    for c, col in zip(r.coeffs, cols):
                        acc = acc * (c * col)
                    ok &= acc <= r.bound
                elif r.kind == "max-weighted-sum":
                    acc = np.zeros(vm.shape[0], dtype=np.int64)
                    for c, col in zip(r.coeffs, cols):
                        acc = acc + c * col
                    ok &= acc <= r.bound
                else:
                    hit = np.ones(vm.shape[0], dtype=bool)
                    for c, col in zip(r.coeffs, cols):
                        hit &= col == c
                    ok &= ~hit
        return ok

    def valid_mask(self, vm: np.ndarray) -> np.ndarray:   # paramspace.py:201-203
        return self.rule_mask(self.rules, vm)

    def encode(self, idx) -> np.ndarray:
        """model.py:88-97: feature = digit / max(count-1, 1), float64."""
        rem = np.asarray(idx, dtype=np.int64).copy()
        out = np.empty((rem.shape[0], len(self.radix)), dtype=np.float64)
        for col in reversed(range(len(self.radix))):
            rem, dig = np.divmod(rem, self.radix[col])
            out[:, col] = dig / max(self.radix[col] - 1, 1)
        return out

    def sample_indices(self, n: int, seed: int) -> np.ndarray:
        """paramspace.py:230-255: prefix-stable PCG64 stream of distinct indices."""
        card = self.card
        if n > card:
            raise ValueError(f"cannot sample {n} distinct configs from {card}")
        rng = make_rng(seed)
        if card <= PERMUTATION_LIMIT:
            return rng.permutation(card)[:n].astype(np.int64)
        seen: set = set()
        out = []
        while len(out) < n:
            for i in rng.integers(0, card, size=4096):
                i = int(i)
                if i not in seen:
                    seen.add(i)
                    out.append(i)
                    if len(out) == n:
                        break
        return np.asarray(out, dtype=np.int64)


def space_from_doc(doc: dict) -> OSpace:
    """Space JSON as written by paramspace.py:347-360."""
    names = [p["name"] for p in doc["params"]]
    pos = {n: i for i, n in enumerate(names)}
    rules = []
    for r in doc.get("rules", ()):
        coeffs = tuple(int(c) for c in r.get("coefficients", ()))
        if not coeffs and r["kind"] != "forbidden-combination":
            coeffs = (1,) * len(r["operands"])           # paramspace.py:74-76
        rules.append(ORule(r["kind"], tuple(pos[o] for o in r["operands"]),
                           coeffs, int(r.get("bound", 0))))
    return OSpace(doc["name"], names, [p["values"] for p in doc["params"]], rules)
