"""Multi-GPU sweep: one process per GPU, contiguous index slices, one NCCL
all-gather of the per-rank top-m.

Rank r of P sweeps [floor(r*C/P), floor((r+1)*C/P)) on its own B200 and keeps
its exact local top-m by (prediction, index). Every element of the global
top-m lies in its own shard's local top-m, so gathering P*m entries
(16 B each: 3.2 KB per rank at m = 200) and re-selecting gives exactly the
single-GPU answer. The merge runs on the device (`mlt_merge_top_m`).

The slice / gather / merge logic is backend-agnostic: CPU tests drive it
over `gloo` with injected local-sweep and merge functions.
"""

from __future__ import annotations

import numpy as np

PAD_IDX = -1


def shard_bounds(card: int, rank: int, world: int) -> tuple[int, int]:
    return card * rank // world, card * (rank + 1) // world


def _device_local(ensemble, space, m, lo, hi):
    from .tuner import top_m_arrays
    return top_m_arrays(ensemble, space, m, begin=lo, end=hi)


def _device_merge(all_idx, all_pred, m):
    """Merge gathered (idx, pred) CUDA tensors on the device."""
    from . import _native as N
    import torch
    out_idx = np.empty(m, dtype=np.int64)
    out_pred = np.empty(m, dtype=np.float64)
    out_n = N.C.c_int64(0)
    dev = all_idx.device.index if all_idx.device.index is not None else torch.cuda.current_device()
    N.check(N.lib().mlt_merge_top_m(N.ctx(dev), N.C.c_void_p(all_idx.data_ptr()), N.C.c_void_p(all_pred.data_ptr()),
                                    all_idx.numel(), m, N.ptr(out_idx, N.C.c_int64), N.ptr(out_pred, N.C.c_double),
                                    N.C.byref(out_n)))
    n = out_n.value
    return out_idx[:n], out_pred[:n]


def gather_top_lists(idx, pred, m: int, group=None):
    """All-gather every rank's (index, prediction) top-m list in ONE collective:
    a per-rank int64 record [m indices | m prediction bit patterns], padded with
    index -1 / +inf. Returns the concatenated (indices, predictions) tensors
    (on the GPU for NCCL, on the CPU for gloo)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    rec = torch.empty(2 * m, dtype=torch.int64)
    rec[:m] = PAD_IDX
    rec[m:] = torch.tensor([float("inf")], dtype=torch.float64).view(torch.int64)
    n = len(idx)
    rec[:n] = torch.from_numpy(np.asarray(idx, dtype=np.int64))
    rec[m:m + n] = torch.from_numpy(np.asarray(pred, dtype=np.float64).view(np.int64))
    rec = rec.to(dev)
    out = torch.empty(world * 2 * m, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(out, rec, group=group)
    out = out.view(world, 2, m)
    return out[:, 0, :].reshape(-1).contiguous(), out[:, 1, :].reshape(-1).contiguous().view(torch.float64)


def _record_from_host(idx, pred, m, dev):
    """A host (index, prediction) list as an mlt_plan_top_m_record record."""
    import torch
    rec = torch.empty(2 * m + 1, dtype=torch.int64)
    rec[:m] = PAD_IDX
    rec[m:2 * m] = torch.tensor([float("inf")], dtype=torch.float64).view(torch.int64)
    n = len(idx)
    rec[:n] = torch.from_numpy(np.asarray(idx, dtype=np.int64))
    rec[m:m + n] = torch.from_numpy(np.asarray(pred, dtype=np.float64).view(np.int64))
    rec[2 * m] = 0
    return rec.to(dev)


def records_protocol(rank: int, world: int, m: int, first_record, gather, merge, redo_record):
    """The exchange of the sharded step, backend- and device-agnostic (CPU
    tests drive it over gloo with numpy records):
      rec = first_record()            this rank's (2m+1)-int64 record
      out = gather(rec)               all ranks' records, (world*(2m+1),)
      idx, pred, status = merge(out)  global top-m, OR of the status words
    A nonzero status means some shard's fast path could not finish (guard
    band overflow): every rank sees the same gathered statuses, the ranks
    whose own status is set rebuild their record with `redo_record()` (the
    exact path), and all ranks gather and merge once more."""
    rec = first_record()
    for attempt in range(2):
        out = gather(rec)
        idx, pred, status = merge(out)
        if status == 0:
            return idx, pred
        if attempt == 1:
            raise RuntimeError("sharded top-m: a shard stayed unresolved after the exact redo")
        mine = int(np.asarray(out.reshape(world, 2 * m + 1)[rank, 2 * m].tolist()))
        if mine != 0:
            rec = redo_record()
    raise AssertionError("unreachable")


def top_m_arrays_records(ensemble, space, m: int, group=None, plan=None):
    """The device-resident sharded step: every rank enqueues its
    shard's top-m straight into a device record (`mlt_plan_top_m_record`, no
    host round trip), ONE all-gather moves the (2m+1)-int64 records (NCCL:
    device to device, ordered on the caller's stream), and `mlt_merge_records`
    sorts the P*m entries on the device with one host wait for the result
    (`records_protocol` handles a shard whose guard band overflowed)."""
    import torch
    import torch.distributed as dist
    from . import _native as N
    if m < 1:
        raise ValueError("m must be >= 1")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.cuda.current_device()
    cdev = torch.device("cuda", dev)
    lo, hi = shard_bounds(space.cardinality(), rank, world)
    plan = plan or N.plan(space, ensemble, dev)

    def first_record():
        rec = torch.empty(2 * m + 1, dtype=torch.int64, device=cdev)
        N.check(N.lib().mlt_plan_top_m_record(plan.h, int(m), lo, hi, N.C.c_void_p(rec.data_ptr())),
                "mlt_plan_top_m_record")
        return rec

    def gather(rec):
        send = rec if nccl else rec.cpu()          # gloo: functional runs only
        out = torch.empty(world * (2 * m + 1), dtype=torch.int64, device=send.device)
        dist.all_gather_into_tensor(out, send, group=group)
        return out if nccl else out.to(cdev)

    def merge(out):
        oi, op = np.empty(m, np.int64), np.empty(m, np.float64)
        on, ost = N.C.c_int64(0), N.C.c_int64(0)
        N.check(N.lib().mlt_merge_records(N.ctx(dev), N.C.c_void_p(out.data_ptr()), world, int(m),
                                          N.ptr(oi, N.C.c_int64), N.ptr(op, N.C.c_double), N.C.byref(on),
                                          N.C.byref(ost)), "mlt_merge_records")
        return oi[:on.value], op[:on.value], ost.value

    def redo_record():
        li, lp = np.empty(m, np.int64), np.empty(m, np.float64)
        ln, st = N.C.c_int64(0), N.MltSweepStats()
        N.check(N.lib().mlt_plan_top_m(plan.h, int(m), lo, hi, N.ptr(li, N.C.c_int64), N.ptr(lp, N.C.c_double),
                                       N.C.byref(ln), N.C.byref(st)), "mlt_plan_top_m")
        return _record_from_host(li[:ln.value], lp[:ln.value], m, cdev)

    with N.on_stream(dev, torch.cuda.current_stream().cuda_stream):
        return records_protocol(rank, world, m, first_record, gather, merge, redo_record)


def top_m_arrays_sharded(ensemble, space, m: int, group=None, local_fn=None, merge_fn=None):
    """Sharded top-m over the whole space; identical result on every rank.
    Without injected local/merge functions (CPU tests inject the oracle) this
    is the device-resident record path, `top_m_arrays_records`."""
    import torch.distributed as dist
    if m < 1:
        raise ValueError("m must be >= 1")
    if local_fn is None and merge_fn is None:
        return top_m_arrays_records(ensemble, space, m, group)
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    lo, hi = shard_bounds(space.cardinality(), rank, world)
    idx, pred = (local_fn or _device_local)(ensemble, space, m, lo, hi)
    gi, gp = gather_top_lists(idx, pred, m, group)
    if merge_fn is not None:
        return merge_fn(gi.cpu().numpy(), gp.cpu().numpy(), m)
    if not gi.is_cuda:          # CPU-side collective (gloo): the merge still runs on this rank's B200
        gi, gp = gi.cuda(), gp.cuda()
    return _device_merge(gi, gp, m)


def top_m_predicted(ensemble, space, m: int, sweep_cap=None, seed: int = 0, group=None):
    """Drop-in for tuner.top_m_predicted across the ranks of `group`
    (sweep_cap subsets are small: they run on each rank's device unsharded)."""
    from .tuner import configs_of, top_m_predicted as single
    if sweep_cap is not None and space.cardinality() > sweep_cap:
        return single(ensemble, space, m, sweep_cap, seed)
    idx, pred = top_m_arrays_sharded(ensemble, space, m, group)
    return list(zip(configs_of(space, idx), np.asarray(pred, dtype=np.float64).tolist()))


def top_m_arrays_multi_device(ensemble, space, m: int, devices, begin: int = 0, end: int | None = None,
                              indices=None, with_stats: bool = False):
    """Single-process multi-GPU top-m (`mlt_top_m_multi`): one shard per entry
    of `devices`, swept concurrently from host threads inside the library,
    merged by (prediction, index). The result equals `tuner.top_m_arrays` over
    the same slice / index list. A device listed twice gets a second context."""
    from . import _native as N
    if m < 1:
        raise ValueError("m must be >= 1")
    devs = [int(d) for d in devices]
    if not devs:
        raise ValueError("need at least one device")
    seen = {}
    ctxs = []
    for d in devs:
        ctxs.append(N.extra_ctx(d, seen.get(d, 0)))
        seen[d] = seen.get(d, 0) + 1
    arr = (N.C.c_void_p * len(ctxs))(*[c.value for c in ctxs])
    ps, pe = N.packed(space, "space"), N.packed(ensemble, "ensemble")
    end = ps.card if end is None else int(end)
    out_idx = np.empty(m, dtype=np.int64)
    out_pred = np.empty(m, dtype=np.float64)
    out_n = N.C.c_int64(0)
    st = N.MltSweepStats()
    if indices is not None:
        lst = np.ascontiguousarray(indices, dtype=np.int64)
        lp, ln = N.ptr(lst, N.C.c_int64), lst.shape[0]
    else:
        lp, ln = None, 0
    N.check(N.lib().mlt_top_m_multi(arr, len(ctxs), N.C.byref(ps.c), N.C.byref(pe.c), int(m), int(begin), end,
                                    lp, ln, N.ptr(out_idx, N.C.c_int64), N.ptr(out_pred, N.C.c_double),
                                    N.C.byref(out_n), N.C.byref(st)), "mlt_top_m_multi")
    n = out_n.value
    res = (out_idx[:n].copy(), out_pred[:n].copy())
    return res + (st.as_dict(),) if with_stats else res


def exhaustive_best_sharded(runner, space, group=None, repetitions=None, local_fn=None):
    """Exhaustive search (tuner.py:191-224) over the ranks of `group`: rank r
    runs the fused device search (`runner.exhaustive_best`) on its slice, one
    all-gather moves 4 numbers per rank (best time, best index, valid count),
    and every rank picks the (time, index) minimum — identical to the
    single-GPU search. Returns (best index or -1, best time, total valid)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    lo, hi = shard_bounds(space.cardinality(), rank, world)
    if local_fn is not None:
        fn = local_fn
    elif hasattr(runner, "exhaustive_best"):
        fn = lambda a, b: runner.exhaustive_best(a, b, repetitions)   # noqa: E731
    else:
        fn = lambda a, b: _measured_slice_best(runner, space, a, b, repetitions)   # noqa: E731
    i, t, nv, _ = fn(lo, hi)
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    mine = torch.tensor([t if i >= 0 else float("inf"), float(i), float(nv)], dtype=torch.float64, device=dev)
    allv = torch.empty(world * 3, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(allv, mine, group=group)
    v = allv.cpu().numpy().reshape(world, 3)
    total = int(v[:, 2].sum())
    ok = v[:, 1] >= 0
    if not ok.any():
        return -1, float("nan"), total
    cand = sorted((float(tt), int(ii)) for tt, ii in zip(v[ok, 0], v[ok, 1]))
    return cand[0][1], cand[0][0], total


def _measured_slice_best(runner, space, lo, hi, repetitions=None, chunk=1 << 17):
    """Minimum (time, index) over the statically valid configurations of
    [lo, hi) measured through `runner.measured_times` (each rank measures its
    own slice on its own device: the sharded ground truth of SURVEY §8(e))."""
    reps = getattr(runner, "default_repetitions", 1) if repetitions is None else repetitions
    best, nv = None, 0
    for s in range(lo, hi, chunk):
        idx = np.arange(s, min(s + chunk, hi), dtype=np.int64)
        if getattr(space, "rules", ()):
            idx = idx[space.valid_mask_indices(idx)] if hasattr(space, "valid_mask_indices") else \
                idx[space.static_valid_mask(space.decode_indices(idx))]
        if idx.size == 0:
            continue
        times, ok = runner.measured_times(idx, reps)
        nv += int(np.count_nonzero(ok))
        if not ok.any():
            continue
        p = int(np.nanargmin(np.where(ok, times, np.nan)))
        key = (float(times[p]), int(idx[p]))
        if best is None or key < best:
            best = key
    if best is None:
        return -1, float("nan"), nv, 0
    return best[1], best[0], nv, 0


def exhaustive_search(space, runner, group=None):
    """Drop-in for tuner.exhaustive_search across ranks: each rank searches its
    contiguous slice (the fused device search for the surrogate, chunked
    `measured_times` for a hardware runner such as the B200 benchmark kernels)
    and one all-gather of 3 numbers per rank picks the global (time, index)
    minimum. Runners with neither method take the single-rank path."""
    from . import errors
    from .tuner import exhaustive_search as single
    if not hasattr(runner, "exhaustive_best") and not hasattr(runner, "measured_times"):
        return single(space, runner)
    i, t, _ = exhaustive_best_sharded(runner, space, group)
    if i < 0:
        raise errors.active["EmptySpaceError"](f"space {space.name!r} has no valid configuration")
    return space.config_at(i), t
