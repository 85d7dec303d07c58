"""Parameter spaces — the API surface of `mltune.paramspace`
(/root/reference/pkg/src/mltune/paramspace.py) with the bulk operations on
the B200.

A space is an ordered list of integer-valued parameters; configuration
indices are mixed radix with the LAST parameter fastest (paramspace.py:149-158).
Scalar helpers (`config_at`, `index_of`) stay on the host; the vectorised
`decode_indices` / `valid_mask_indices` / `static_valid_mask` run as CUDA
kernels through the C ABI (A1/A2 of SURVEY §8).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _native as N
from .errors import ConfigMismatchError, ParseError

Configuration = tuple
BUILTIN_SPACE_NAMES = ("convolution", "raycasting", "stereo")
RULE_KINDS = ("max-product", "max-weighted-sum", "forbidden-combination")
PERMUTATION_LIMIT = 1 << 22   # sampling switches to rejection above this (paramspace.py:35)


def make_rng(*parts: int) -> np.random.Generator:
    """PCG64 from SeedSequence(parts mod 2^64) — the reference stream (rng.py:15-22)."""
    return np.random.default_rng(np.random.SeedSequence([int(p) & ((1 << 64) - 1) for p in parts]))


def derive_seed(*parts: int) -> int:
    """rng.py:25-27."""
    ss = np.random.SeedSequence([int(p) & ((1 << 64) - 1) for p in parts])
    return int(ss.generate_state(1, dtype=np.uint64)[0])


@dataclass(frozen=True)
class ParamDef:
    name: str
    values: tuple

    def __post_init__(self):
        vals = tuple(int(v) for v in self.values)
        object.__setattr__(self, "values", vals)
        if not vals:
            raise ValueError(f"parameter {self.name!r} has an empty value list")
        if len(set(vals)) != len(vals):
            raise ValueError(f"parameter {self.name!r} has duplicate values")


@dataclass(frozen=True)
class ValidityRule:
    """max-product: prod(c*v) <= bound; max-weighted-sum: sum(c*v) <= bound;
    forbidden-combination: invalid when every operand equals its coefficient."""
    kind: str
    operands: tuple
    coefficients: tuple = ()
    bound: int = 0

    def __post_init__(self):
        if self.kind not in RULE_KINDS:
            raise ValueError(f"unknown rule kind {self.kind!r}")
        ops = tuple(self.operands)
        co = tuple(int(c) for c in self.coefficients)
        if not co and self.kind != "forbidden-combination":
            co = (1,) * len(ops)
        if len(co) != len(ops):
            raise ValueError(f"rule {self.kind} has {len(ops)} operands but {len(co)} coefficients")
        object.__setattr__(self, "operands", ops)
        object.__setattr__(self, "coefficients", co)

    def is_satisfied(self, assignment) -> bool:
        vals = [int(assignment[o]) for o in self.operands]
        mask = 0xFFFFFFFFFFFFFFFF
        if self.kind == "forbidden-combination":
            return any(v != c for v, c in zip(vals, self.coefficients))
        acc = 1 if self.kind == "max-product" else 0
        for c, v in zip(self.coefficients, vals):   # int64 wrap-around like numpy
            acc = (acc * (c * v)) & mask if self.kind == "max-product" else (acc + c * v) & mask
        acc = acc - (1 << 64) if acc >= (1 << 63) else acc
        return acc <= self.bound


@dataclass(frozen=True)
class ParamSpace:
    name: str
    params: tuple
    rules: tuple = ()
    _pos: dict = field(init=False, repr=False, compare=False, hash=False)

    def __post_init__(self):
        object.__setattr__(self, "params", tuple(self.params))
        object.__setattr__(self, "rules", tuple(self.rules))
        names = [p.name for p in self.params]
        if len(set(names)) != len(names):
            raise ValueError(f"space {self.name!r} has duplicate parameter names")
        object.__setattr__(self, "_pos", {n: i for i, n in enumerate(names)})
        for r in self.rules:
            missing = [o for o in r.operands if o not in self._pos]
            if missing:
                raise ValueError(f"rule {r.kind} references unknown parameters {missing}")

    # -- scalar indexing (host) ---------------------------------------------
    def cardinality(self) -> int:
        return math.prod(len(p.values) for p in self.params)

    def param_names(self) -> list:
        return [p.name for p in self.params]

    def param_index(self, name: str) -> int:
        try:
            return self._pos[name]
        except KeyError:
            raise KeyError(f"no parameter {name!r} in space {self.name!r}") from None

    def config_at(self, index: int) -> Configuration:
        card = self.cardinality()
        if not 0 <= index < card:
            raise IndexError(f"index {index} out of range for {card} configurations")
        digits = []
        for p in reversed(self.params):
            index, d = divmod(index, len(p.values))
            digits.append(p.values[d])
        return tuple(reversed(digits))

    def configs_at(self, indices) -> list:
        """`[config_at(i) for i in indices]`, decoded column-wise with numpy
        (the per-index Python loop was the largest host cost of a top-m call)."""
        idx = np.asarray(indices, dtype=np.int64).reshape(-1)
        if idx.size == 0:
            return []
        card = self.cardinality()
        lo, hi = int(idx.min()), int(idx.max())
        if lo < 0 or hi >= card:
            raise IndexError(f"index {lo if lo < 0 else hi} out of range for {card} configurations")
        dec = self.__dict__.get("_decode")
        if dec is None:   # (value table, strides, radices, columns): the space is immutable
            radix = [len(p.values) for p in self.params]
            table = np.zeros((len(radix), max(radix)), dtype=np.int64)
            try:
                for col, p in enumerate(self.params):
                    table[col, :radix[col]] = p.values
            except OverflowError:   # a parameter value beyond int64: decode one by one
                table = None
            strides = np.ones(len(radix), dtype=np.int64)
            for col in range(len(radix) - 2, -1, -1):
                strides[col] = strides[col + 1] * radix[col + 1]
            dec = (table, strides[None, :], np.asarray(radix, dtype=np.int64)[None, :],
                   np.arange(len(radix))[None, :])
            object.__setattr__(self, "_decode", dec)
        table, strides, radix, cols = dec
        if table is None:
            return [self.config_at(i) for i in idx.tolist()]
        vals = table[cols, (idx[:, None] // strides) % radix]
        return list(map(tuple, vals.tolist()))

    def validate_config(self, config) -> None:
        if len(config) != len(self.params):
            raise ConfigMismatchError(f"configuration has {len(config)} values, space {self.name!r} "
                                      f"has {len(self.params)} parameters")
        for p, v in zip(self.params, config):
            if v not in p.values:
                raise ConfigMismatchError(f"value {v} is not admissible for parameter {p.name!r}")

    def index_of(self, config) -> int:
        self.validate_config(config)
        idx = 0
        for p, v in zip(self.params, config):
            idx = idx * len(p.values) + p.values.index(v)
        return idx

    def to_dict(self, config) -> dict:
        return dict(zip(self.param_names(), config))

    def is_statically_valid(self, config) -> bool:
        self.validate_config(config)
        a = self.to_dict(config)
        return all(r.is_satisfied(a) for r in self.rules)

    # -- vectorised (B200) ----------------------------------------------------
    def decode_indices(self, indices) -> np.ndarray:
        """(n,) indices -> (n, P) int64 values on the device (paramspace.py:184-193)."""
        return decode_indices(self, indices)

    def valid_mask_indices(self, indices) -> np.ndarray:
        return valid_mask_indices(self, indices)

    def static_valid_mask(self, value_matrix) -> np.ndarray:
        """Vectorised rule check over a value matrix (paramspace.py:201-203):
        values are mapped back to indices (host packing), the rules run on the device."""
        vm = np.asarray(value_matrix, dtype=np.int64)
        return valid_mask_indices(self, self.indices_of_values(vm))

    def indices_of_values(self, vm: np.ndarray) -> np.ndarray:
        idx = np.zeros(vm.shape[0], dtype=np.int64)
        for col, p in enumerate(self.params):
            vals = np.asarray(p.values, dtype=np.int64)
            order = np.argsort(vals)
            pos = np.searchsorted(vals[order], vm[:, col])
            pos = np.clip(pos, 0, len(vals) - 1)
            if not np.array_equal(vals[order][pos], vm[:, col]):
                raise ConfigMismatchError(f"value matrix holds a value not admissible for {p.name!r}")
            idx = idx * len(vals) + order[pos]
        return idx

    # -- sampling (host RNG: must reproduce the reference stream) ---------------
    def sample_indices(self, n: int, seed: int) -> np.ndarray:
        card = self.cardinality()
        if n > card:
            raise ValueError(f"cannot sample {n} distinct configs from {card}")
        rng = make_rng(seed)
        if card <= PERMUTATION_LIMIT:
            return rng.permutation(card)[:n].astype(np.int64)
        seen, out = set(), []
        while len(out) < n:
            for i in rng.integers(0, card, size=4096).tolist():
                if i not in seen:
                    seen.add(i)
                    out.append(i)
                    if len(out) == n:
                        break
        return np.asarray(out, dtype=np.int64)

    def sample_random(self, n: int, seed: int) -> list:
        return self.configs_at(self.sample_indices(n, seed))

    def iter_random_indices(self, seed: int):
        """Prefix-stable seeded stream of distinct indices (paramspace.py:237-255):
        a PCG64 permutation up to 2^22 configurations, else rejection sampling
        in batches of 4096 against a seen-set."""
        card = self.cardinality()
        rng = make_rng(seed)
        if card <= PERMUTATION_LIMIT:
            yield from (int(i) for i in rng.permutation(card))
            return
        seen = set()
        while len(seen) < card:
            for i in rng.integers(0, card, size=4096).tolist():
                if i not in seen:
                    seen.add(i)
                    yield i


def decode_indices(space, indices, device=None) -> np.ndarray:
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    pk = N.packed(space, "space")
    out = np.empty((idx.shape[0], pk.radix.shape[0]), dtype=np.int64)
    if idx.shape[0]:
        N.check(N.lib().mlt_decode(N.ctx(device), N.C.byref(pk.c), N.ptr(idx, N.C.c_int64), idx.shape[0],
                                   N.ptr(out, N.C.c_int64)))
    return out


def valid_mask_indices(space, indices, device=None) -> np.ndarray:
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    pk = N.packed(space, "space")
    out = np.empty(idx.shape[0], dtype=np.uint8)
    if idx.shape[0]:
        N.check(N.lib().mlt_valid_mask(N.ctx(device), N.C.byref(pk.c), N.ptr(idx, N.C.c_int64), idx.shape[0],
                                       N.ptr(out, N.C.c_uint8)))
    return out.astype(bool)


# -- builtin spaces (paramspace.py:283-334: the paper's Table 2 knobs) ------------
_POW2 = (1, 2, 4, 8, 16, 32, 64, 128)
_FLAGS = {
    "convolution": ["use_image", "use_local", "padding", "interleaved", "unroll"],
    "raycasting": ["img_data", "img_transfer", "local_transfer", "const_transfer", "interleaved"],
    "stereo": ["img_left", "img_right", "local_left", "local_right"],
}
_EXTRA = {
    "convolution": [],
    "raycasting": [("unroll_ray", (1, 2, 4, 8, 16))],
    "stereo": [("unroll_disparity", (1, 2, 4, 8)), ("unroll_diff_x", (1, 2, 4)), ("unroll_diff_y", (1, 2, 4))],
}


def builtin_space(name: str) -> ParamSpace:
    if name not in BUILTIN_SPACE_NAMES:
        raise ValueError(f"unknown built-in space {name!r}; expected one of {BUILTIN_SPACE_NAMES}")
    ps = [ParamDef(n, _POW2) for n in ("wg_x", "wg_y", "ppt_x", "ppt_y")]
    ps += [ParamDef(n, (0, 1)) for n in _FLAGS[name]]
    ps += [ParamDef(n, v) for n, v in _EXTRA[name]]
    return ParamSpace(name, tuple(ps))


def space_to_json(space) -> dict:
    return {"name": space.name,
            "params": [{"name": p.name, "values": list(p.values)} for p in space.params],
            "rules": [{"kind": r.kind, "operands": list(r.operands), "coefficients": list(r.coefficients),
                       "bound": r.bound} for r in space.rules]}


def space_from_json(doc: dict, source="<json>") -> ParamSpace:
    try:
        params = tuple(ParamDef(p["name"], tuple(p["values"])) for p in doc["params"])
        rules = tuple(ValidityRule(r["kind"], tuple(r["operands"]), tuple(r.get("coefficients", ())),
                                   int(r.get("bound", 0))) for r in doc.get("rules", ()))
        return ParamSpace(doc["name"], params, rules)
    except (KeyError, TypeError, ValueError) as exc:
        raise ParseError(f"bad space definition: {exc}", path=source) from exc


def load_space(path) -> ParamSpace:
    path = Path(path)
    try:
        doc = json.loads(path.read_text())
    except json.JSONDecodeError as exc:
        raise ParseError(f"not valid JSON: {exc}", path=path) from exc
    return space_from_json(doc, source=path)


def save_space(space, path) -> None:
    Path(path).write_text(json.dumps(space_to_json(space), indent=2) + "\n")
