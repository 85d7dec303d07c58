"""ctypes binding of libmltune_b200.so (the C ABI in include/mltune_b200.h).

Packs duck-typed space / ensemble objects — this package's own or the
reference `mltune`'s — into the plain C descriptors, owns one library context
per CUDA device (the library serialises calls on a context, so one context
can be shared across threads), and maps native status codes to the tuner's
exceptions.
Nothing here computes: every numeric entry point runs on the B200. If the
library or the device is missing, calls raise NativeUnavailableError.
"""

from __future__ import annotations

import atexit
import ctypes as C
import os
import threading
import weakref
from pathlib import Path

import numpy as np

from . import errors

_LIB_PATH = Path(os.environ.get("MLTUNE_B200_LIB", Path(__file__).resolve().parent / "libmltune_b200.so"))

MLT_OK, MLT_EINVAL, MLT_EMISMATCH, MLT_EDATA, MLT_EDIVERGED, MLT_ECUDA, MLT_EINTERNAL = 0, -1, -2, -3, -4, -5, -6
(MLT_OPT_PATH, MLT_OPT_GROUP, MLT_OPT_CAND_CAP, MLT_OPT_PRUNE, MLT_OPT_CHUNK, MLT_OPT_TABLE_CACHE,
 MLT_OPT_HALF_ITEMS, MLT_OPT_TAIL_SPLIT) = 1, 2, 3, 4, 5, 6, 7, 8
RULE_KIND = {"max-product": 0, "max-weighted-sum": 1, "forbidden-combination": 2}

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


class MltSpace(C.Structure):
    _fields_ = [("n_params", C.c_int32), ("radix", _i32p), ("values", _i64p), ("n_rules", C.c_int32),
                ("rule_kind", _i32p), ("rule_nops", _i32p), ("rule_pos", _i32p), ("rule_coeff", _i64p),
                ("rule_bound", _i64p)]


class MltEnsemble(C.Structure):
    _fields_ = [("k", C.c_int32), ("d", C.c_int32), ("h", C.c_int32), ("counts", _i32p), ("w1", _f64p),
                ("b1", _f64p), ("w2", _f64p), ("b2", _f64p), ("mean", _f64p), ("std", _f64p)]


class MltSweepStats(C.Structure):
    _fields_ = [("configs", C.c_int64), ("candidates", C.c_int64), ("path", C.c_int32), ("group", C.c_int32),
                ("delta", C.c_double), ("sweep_ms", C.c_float), ("total_ms", C.c_float),
                ("launches", C.c_int32), ("split", C.c_int32), ("raw_candidates", C.c_int64),
                ("evaluated_frac", C.c_double)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


class MltTrainDesc(C.Structure):
    _fields_ = [("k", C.c_int32), ("d", C.c_int32), ("h", C.c_int32), ("epochs", C.c_int32),
                ("batch_size", C.c_int32), ("learning_rate", C.c_double), ("momentum", C.c_double),
                ("n_rows", C.c_int64), ("x", _f64p), ("t", _f64p), ("rows", _i32p), ("n_m", _i32p),
                ("init_w1", _f64p), ("init_w2", _f64p), ("perms", _i32p)]


class MltSurrogate(C.Structure):
    _fields_ = [("base_time", C.c_double), ("n_terms", C.c_int32), ("term_nparams", _i32p), ("term_pos", _i32p),
                ("term_match", _i64p), ("term_factor", _f64p), ("log_sigma", C.c_double), ("seed", C.c_uint64),
                ("n_rules", C.c_int32), ("rule_kind", _i32p), ("rule_nops", _i32p), ("rule_pos", _i32p),
                ("rule_coeff", _i64p), ("rule_bound", _i64p)]


# (name, restype, argtypes) of every exported entry point of the header.
_SIGNATURES = [
    ("mlt_abi_version", C.c_int, []),
    ("mlt_last_error", C.c_char_p, []),
    ("mlt_ctx_create", C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    ("mlt_ctx_destroy", C.c_int, [C.c_void_p]),
    ("mlt_ctx_set_stream", C.c_int, [C.c_void_p, C.c_void_p]),
    ("mlt_ctx_set_profiling", C.c_int, [C.c_void_p, C.c_int]),
    ("mlt_ctx_launches", C.c_int64, [C.c_void_p]),
    ("mlt_ctx_set_option", C.c_int, [C.c_void_p, C.c_int, C.c_int64]),
    ("mlt_decode", C.c_int, [C.c_void_p, C.POINTER(MltSpace), _i64p, C.c_int64, _i64p]),
    ("mlt_valid_mask", C.c_int, [C.c_void_p, C.POINTER(MltSpace), _i64p, C.c_int64, _u8p]),
    ("mlt_encode", C.c_int, [C.c_void_p, _i32p, C.c_int32, _i64p, C.c_int64, _f64p]),
    ("mlt_predict_indices", C.c_int, [C.c_void_p, C.POINTER(MltEnsemble), _i64p, C.c_int64, _f64p]),
    ("mlt_predict_features", C.c_int, [C.c_void_p, C.POINTER(MltEnsemble), _f64p, C.c_int64, _f64p]),
    ("mlt_member_outputs", C.c_int, [C.c_void_p, C.POINTER(MltEnsemble), _f64p, C.c_int64, _f64p]),
    ("mlt_top_m", C.c_int, [C.c_void_p, C.POINTER(MltSpace), C.POINTER(MltEnsemble), C.c_int64, C.c_int64,
                            C.c_int64, _i64p, C.c_int64, _i64p, _f64p, _i64p, C.POINTER(MltSweepStats)]),
    ("mlt_top_m_multi", C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.POINTER(MltSpace), C.POINTER(MltEnsemble),
                                  C.c_int64, C.c_int64, C.c_int64, _i64p, C.c_int64, _i64p, _f64p, _i64p,
                                  C.POINTER(MltSweepStats)]),
    ("mlt_plan_create", C.c_int, [C.c_void_p, C.POINTER(MltSpace), C.POINTER(MltEnsemble), C.POINTER(C.c_void_p)]),
    ("mlt_plan_top_m", C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, _i64p, _f64p, _i64p,
                                 C.POINTER(MltSweepStats)]),
    ("mlt_plan_destroy", C.c_int, [C.c_void_p]),
    ("mlt_merge_top_m", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, _i64p, _f64p, _i64p]),
    ("mlt_plan_top_m_record", C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p]),
    ("mlt_merge_records", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, _i64p, _f64p, _i64p, _i64p]),
    ("mlt_train_members", C.c_int, [C.c_void_p, C.POINTER(MltTrainDesc), _f64p, _f64p, _f64p, _f64p, _f64p,
                                     _f64p, _i32p]),
    ("mlt_format_predictions", C.c_int, [_i64p, _f64p, C.c_int64, C.c_char_p, C.c_int64, _i64p, C.c_int32]),
    ("mlt_host_permutations", C.c_int, [C.POINTER(C.c_void_p), C.c_int32, _i32p, C.c_int32, _i32p, C.c_int32]),
    ("mlt_surrogate_times", C.c_int, [C.c_void_p, C.POINTER(MltSpace), C.POINTER(MltSurrogate), _i64p, C.c_int64,
                                      C.c_int32, _f64p, _u8p]),
    ("mlt_surrogate_best", C.c_int, [C.c_void_p, C.POINTER(MltSpace), C.POINTER(MltSurrogate), C.c_int64, C.c_int64,
                                     C.c_int32, C.c_double, _i64p, _f64p, _i64p, _i64p]),
    ("mlt_convbench_create", C.c_int, [C.c_int, C.c_int32, C.c_int32, C.POINTER(C.c_float), C.c_uint64,
                                       C.POINTER(C.c_void_p)]),
    ("mlt_convbench_destroy", C.c_int, [C.c_void_p]),
    ("mlt_convbench_run", C.c_int, [C.c_void_p, _i32p, C.c_int32, _f64p, _i32p]),
    ("mlt_convbench_output", C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    ("mlt_convbench_input", C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    ("mlt_convbench_last_error", C.c_char_p, []),
    ("mlt_stereobench_create", C.c_int, [C.c_int, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _u8p, _u8p,
                                         C.c_uint64, C.POINTER(C.c_void_p)]),
    ("mlt_stereobench_destroy", C.c_int, [C.c_void_p]),
    ("mlt_stereobench_run", C.c_int, [C.c_void_p, _i32p, C.c_int32, _f64p, _i32p]),
    ("mlt_stereobench_output", C.c_int, [C.c_void_p, _u8p]),
    ("mlt_stereobench_set_budget", C.c_int, [C.c_void_p, C.c_uint64]),
    ("mlt_stereobench_input", C.c_int, [C.c_void_p, _u8p, _u8p]),
    ("mlt_stereobench_last_error", C.c_char_p, []),
    ("mlt_raybench_create", C.c_int, [C.c_int, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _u8p,
                                      C.POINTER(C.c_float), C.c_uint64, C.POINTER(C.c_void_p)]),
    ("mlt_raybench_destroy", C.c_int, [C.c_void_p]),
    ("mlt_raybench_run", C.c_int, [C.c_void_p, _i32p, C.c_int32, _f64p, _i32p]),
    ("mlt_raybench_output", C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    ("mlt_raybench_set_budget", C.c_int, [C.c_void_p, C.c_uint64]),
    ("mlt_raybench_volume", C.c_int, [C.c_void_p, _u8p]),
    ("mlt_raybench_transfer", C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    ("mlt_raybench_camera", C.c_int, [C.c_void_p, C.POINTER(C.c_float)]),
    ("mlt_raybench_last_error", C.c_char_p, []),
]
EXPORTS = tuple(name for name, _, _ in _SIGNATURES)

ABI_VERSION = 1      # MLT_ABI_VERSION of include/mltune_b200.h this binding's structs follow

_lib = None
_lib_lock = threading.Lock()
_ctx_lock = threading.Lock()
_ctxs: dict[int, C.c_void_p] = {}


def lib():
    """Load the in-tree library (fails loudly; there is no fallback)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise errors.NativeUnavailableError(
                    f"{_LIB_PATH} is not built; run __graft_entry__.build() (nvcc, sm_100a)")
            h = C.CDLL(str(_LIB_PATH))
            for name, res, args in _SIGNATURES:
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            if h.mlt_abi_version() != ABI_VERSION:
                raise errors.NativeUnavailableError(
                    f"{_LIB_PATH} has ABI version {h.mlt_abi_version()}, this binding expects {ABI_VERSION}; "
                    "rebuild it with __graft_entry__.build()")
            _lib = h
    return _lib


def last_error() -> str:
    return (lib().mlt_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str = "", epoch: int | None = None):
    if rc == MLT_OK:
        return
    msg = last_error() or what
    if rc == MLT_EINVAL:
        raise ValueError(msg)
    if rc == MLT_EMISMATCH:
        raise errors.active["ConfigMismatchError"](msg)
    if rc == MLT_EDATA:
        raise errors.active["InsufficientDataError"](msg)
    if rc == MLT_EDIVERGED:
        raise errors.active["DivergenceError"](msg, epoch=epoch if epoch is not None else -1)
    if rc == MLT_ECUDA:
        raise errors.NativeUnavailableError(msg)
    raise RuntimeError(f"libmltune_b200 internal error: {msg}")


def default_device() -> int:
    env = os.environ.get("MLTUNE_B200_DEVICE")
    if env is not None:
        return int(env)
    try:
        import torch
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            return torch.cuda.current_device()
    except Exception:  # torch is optional plumbing
        pass
    return 0


def ctx(device: int | None = None) -> C.c_void_p:
    """The library context of `device` (created on first use)."""
    dev = default_device() if device is None else int(device)
    hit = _ctxs.get(dev)
    if hit is not None:
        return hit
    with _ctx_lock:            # one context per device even under concurrent first use
        if dev not in _ctxs:
            h = C.c_void_p()
            check(lib().mlt_ctx_create(dev, C.byref(h)), "mlt_ctx_create")
            _ctxs[dev] = h
    return _ctxs[dev]


def extra_ctx(device: int, slot: int) -> C.c_void_p:
    """An additional context on `device` (slot >= 1; slot 0 is ctx(device)):
    contexts are not re-entrant, so concurrent work on one device needs one each."""
    if slot == 0:
        return ctx(device)
    key = (int(device), int(slot))
    with _ctx_lock:
        if key not in _ctxs:
            h = C.c_void_p()
            check(lib().mlt_ctx_create(int(device), C.byref(h)), "mlt_ctx_create")
            _ctxs[key] = h
    return _ctxs[key]


class Plan:
    """A resident mlt_plan of one (space, ensemble) on one device: the
    descriptors are uploaded and the factored tables built once, and kept
    while the plan lives (the reference's spaces and ensembles are immutable,
    model.py:262-301, so identity is a sound cache key)."""

    def __init__(self, space, ensemble, device):
        self.device = int(device)
        self.ctx = ctx(self.device)
        self.ps, self.pe = packed(space, "space"), packed(ensemble, "ensemble")
        self.h = C.c_void_p()
        check(lib().mlt_plan_create(self.ctx, C.byref(self.ps.c), C.byref(self.pe.c), C.byref(self.h)),
              "mlt_plan_create")
        _live_plans.add(self)

    def destroy(self):
        if self.h:
            if _lib is not None and _ctxs.get(self.device) is not None:
                _lib.mlt_plan_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        # plans live while anyone holds them: the cache only drops its reference
        try:
            self.destroy()
        except Exception:   # interpreter shutdown: the library may be gone
            pass


_plan_cache: dict[tuple, tuple] = {}
_live_plans: "weakref.WeakSet[Plan]" = weakref.WeakSet()   # shutdown() frees these before the contexts
_PLAN_CACHE_MAX = 8


def plan(space, ensemble, device=None) -> Plan:
    """The cached resident plan of (space, ensemble) on `device` (LRU of
    _PLAN_CACHE_MAX plans; the cache pins both objects so ids stay unique)."""
    dev = default_device() if device is None else int(device)
    key = (dev, id(space), id(ensemble))
    with _ctx_lock:
        hit = _plan_cache.pop(key, None)
        if hit is not None and hit[0] is space and hit[1] is ensemble:
            _plan_cache[key] = hit                      # most recently used last
            return hit[2]
    p = Plan(space, ensemble, dev)
    with _ctx_lock:
        _plan_cache[key] = (space, ensemble, p)
        while len(_plan_cache) > _PLAN_CACHE_MAX:
            _plan_cache.pop(next(iter(_plan_cache)))   # destroyed once no caller holds it
    return p


def clear_plans() -> None:
    """Drop every cached plan (each is destroyed once no caller holds it)."""
    with _ctx_lock:
        _plan_cache.clear()


CUDA_STREAM_LEGACY = 1   # cudaStreamLegacy: the legacy default stream as an explicit handle


def stream_handle(torch_stream) -> int:
    """A torch stream as a handle for mlt_ctx_set_stream. torch's default
    stream reports handle 0, which mlt_ctx_set_stream reads as "the library's
    own (non-blocking) stream"; pass cudaStreamLegacy instead so the library's
    work really orders against torch's kernels and events."""
    return int(torch_stream.cuda_stream) or CUDA_STREAM_LEGACY


class on_stream:
    """Run a context's work on a CUDA stream (a torch stream's handle) for the
    duration of a `with` block, so device results order against collectives
    and kernels the caller enqueues on that stream; the previous stream is
    restored afterwards."""
    _current: dict[int, int] = {}

    def __init__(self, device: int, stream_handle: int):
        # handle 0 from torch is its legacy default stream, not "no stream"
        self.device, self.handle = int(device), int(stream_handle) or CUDA_STREAM_LEGACY

    def __enter__(self):
        self.prev = on_stream._current.get(self.device, 0)
        check(lib().mlt_ctx_set_stream(ctx(self.device), C.c_void_p(self.handle or None)), "mlt_ctx_set_stream")
        on_stream._current[self.device] = self.handle
        return self

    def __exit__(self, *exc):
        lib().mlt_ctx_set_stream(ctx(self.device), C.c_void_p(self.prev or None))
        on_stream._current[self.device] = self.prev


def shutdown() -> None:
    """Destroy every context (workspaces, pinned staging, streams). Registered
    with atexit so a process ends with the library's device memory released
    (compute-sanitizer's leak check sees no leftovers); ctx() after this
    creates fresh contexts."""
    with _ctx_lock:
        _plan_cache.clear()
    for p in list(_live_plans):   # cached or still held: before their contexts go away
        p.destroy()
    with _ctx_lock:
        items = list(_ctxs.items())
        _ctxs.clear()
    if _lib is None:
        return
    for _, h in items:
        _lib.mlt_ctx_destroy(h)


atexit.register(shutdown)


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


# ---- descriptor packing ------------------------------------------------------

def pack_rules(rules, pos):
    """ValidityRule-likes (kind, operands, coefficients, bound) -> the five
    mlt_space rule arrays (paramspace.py:66-107 semantics; empty coefficients
    mean all ones except for forbidden combinations)."""
    kinds, nops, rpos, coeff, bound = [], [], [], [], []
    for r in rules:
        kind = r["kind"] if isinstance(r, dict) else r.kind
        ops = list(r["operands"] if isinstance(r, dict) else r.operands)
        co = [int(c) for c in (r.get("coefficients", ()) if isinstance(r, dict) else r.coefficients)]
        if not co and kind != "forbidden-combination":
            co = [1] * len(ops)
        if len(co) != len(ops):
            raise ValueError(f"rule {kind} has {len(ops)} operands but {len(co)} coefficients")
        kinds.append(RULE_KIND[kind])
        nops.append(len(ops))
        rpos.extend(pos[o] for o in ops)
        coeff.extend(co)
        bound.append(int(r.get("bound", 0) if isinstance(r, dict) else r.bound))
    return (np.ascontiguousarray(kinds or [0], dtype=np.int32), np.ascontiguousarray(nops or [0], dtype=np.int32),
            np.ascontiguousarray(rpos or [0], dtype=np.int32), np.ascontiguousarray(coeff or [0], dtype=np.int64),
            np.ascontiguousarray(bound or [0], dtype=np.int64))


class PackedSpace:
    """mlt_space over host arrays kept alive by this object."""

    def __init__(self, space):
        params = list(space.params)
        names = [p.name for p in params]
        pos = {n: i for i, n in enumerate(names)}
        self.radix = np.ascontiguousarray([len(p.values) for p in params], dtype=np.int32)
        self.values = np.ascontiguousarray([int(v) for p in params for v in p.values], dtype=np.int64)
        rules = list(getattr(space, "rules", ()))
        self.kind, self.nops, self.rpos, self.coeff, self.bound = pack_rules(rules, pos)
        self.c = MltSpace(len(params), ptr(self.radix, C.c_int32), ptr(self.values, C.c_int64), len(rules),
                          ptr(self.kind, C.c_int32), ptr(self.nops, C.c_int32), ptr(self.rpos, C.c_int32),
                          ptr(self.coeff, C.c_int64), ptr(self.bound, C.c_int64))
        self.card = int(np.prod(self.radix.astype(object)))


class PackedEnsemble:
    """mlt_ensemble over host arrays: [k][h][d] W1, [k][h] b1/w2, [k] b2/mean/std."""

    def __init__(self, ensemble):
        members = list(ensemble.members)
        enc = ensemble.encoder
        self.counts = np.ascontiguousarray([len(vals) for _, vals in enc.params], dtype=np.int32)
        h, d = np.asarray(members[0].weights_hidden).shape
        # np.array over the member list builds each stacked block in one call (C order)
        self.w1 = np.array([m.weights_hidden for m in members], dtype=np.float64)
        self.b1 = np.array([m.biases_hidden for m in members], dtype=np.float64)
        self.w2 = np.array([m.weights_out for m in members], dtype=np.float64)
        self.b2 = np.array([m.bias_out for m in members], dtype=np.float64)
        self.mean = np.array([m.target_mean for m in members], dtype=np.float64)
        self.std = np.array([m.target_std for m in members], dtype=np.float64)
        if self.w1.shape != (len(members), h, d) or self.counts.shape[0] != d:
            raise ValueError("member input dimensions do not match the encoder")
        self.c = MltEnsemble(len(members), d, h, ptr(self.counts, C.c_int32), ptr(self.w1, C.c_double),
                             ptr(self.b1, C.c_double), ptr(self.w2, C.c_double), ptr(self.b2, C.c_double),
                             ptr(self.mean, C.c_double), ptr(self.std, C.c_double))


_pack_cache: dict[int, tuple] = {}


def packed(obj, kind):
    """Cache packed descriptors by object identity (spaces and ensembles are
    immutable in the reference API); the cache pins the object so ids stay unique."""
    key = id(obj)
    hit = _pack_cache.get(key)
    if hit is not None and hit[0] is obj:
        return hit[1]
    pk = PackedSpace(obj) if kind == "space" else PackedEnsemble(obj)
    if len(_pack_cache) > 64:
        _pack_cache.clear()
    _pack_cache[key] = (obj, pk)
    return pk
