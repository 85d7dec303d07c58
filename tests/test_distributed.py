"""Multi-rank sharding logic over `gloo` (world size 2 and 3, CPU): slices
cover the space exactly once, and gather + merge of per-rank top-m equals
the single-process top-m. The per-slice sweep and the merge are injected
(oracle slice sweep, numpy lexsort) so the host logic is tested without a GPU;
on B200s the same code path calls the device sweep and `mlt_merge_top_m`."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, m, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist
    from conftest import CASE_SPACE, oracle_ensemble, oracle_space
    from oracle.tuner import top_m
    from paper_1506_00842_b200.distributed import top_m_arrays_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        osp = oracle_space(CASE_SPACE[case])
        oens = oracle_ensemble(case)

        class SpaceView:           # the product API only needs cardinality() here
            def cardinality(self):
                return osp.card

        def local(ens, space, mm, lo, hi):
            return top_m(oens, osp, mm, begin=lo, end=hi)

        def merge(gi, gp, mm):
            keep = gi >= 0
            gi, gp = gi[keep], gp[keep]
            o = np.lexsort((gi, gp))[:mm]
            return gi[o], gp[o]

        i, p = top_m_arrays_sharded(None, SpaceView(), m, local_fn=local, merge_fn=merge)
        q.put((rank, i.tolist(), p.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_top_m_equals_single_sweep(world):
    from conftest import golden
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, "conv_k1", 200, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = golden("topm_conv_k1.npz")
    for rank, i, p in res:
        assert i == g["m200_i"].tolist(), rank
        assert p == g["m200_p"].tolist()


def test_shard_bounds_partition_the_space():
    from paper_1506_00842_b200.distributed import shard_bounds
    for card in (1, 7, 131072, 100663296):
        for world in (1, 2, 3, 8):
            bounds = [shard_bounds(card, r, world) for r in range(world)]
            assert bounds[0][0] == 0 and bounds[-1][1] == card
            assert all(bounds[r][1] == bounds[r + 1][0] for r in range(world - 1))


def _ex_worker(rank, world, port, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist
    from conftest import oracle_space, surrogates_doc
    from oracle.surrogate import OSurrogate
    from paper_1506_00842_b200.distributed import exhaustive_best_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        osp = oracle_space("convolution")
        ora = OSurrogate(surrogates_doc()["convolution"], osp)

        class SpaceView:
            def cardinality(self):
                return osp.card

        def local(lo, hi):         # the oracle slice search standing in for the device kernel
            idx = np.arange(lo, hi, dtype=np.int64)
            t, ok = ora.measured_times(idx, 1)
            if not ok.any():
                return -1, float("nan"), 0, 0
            tt = np.where(ok, t, np.inf)
            p = int(np.argmin(tt))
            return int(idx[p]), float(tt[p]), int(ok.sum()), 0

        res = exhaustive_best_sharded(None, SpaceView(), local_fn=local)

        class MeasuredRunner:             # a hardware-style runner: measured_times, no fused search
            default_repetitions = 1

            def measured_times(self, idx, reps=1):
                return ora.measured_times(np.asarray(idx), reps)

        class RuleFreeSpace(SpaceView):
            rules = ()

        res2 = exhaustive_best_sharded(MeasuredRunner(), RuleFreeSpace())
        assert res2 == res, (res, res2)
        q.put((rank,) + tuple(res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_exhaustive_equals_single(world):
    """the conv gpu-a optimum is index 88599 — from any shard count."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ex_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, i, t, nv in res:
        assert i == 88599 and abs(t - 0.014444711) < 1e-8 and nv > 0


def _records_worker(rank, world, port, case, m, bad_rank, q):
    """records_protocol over gloo with numpy records: rank `bad_rank` reports a
    guard-band overflow on its first record (status 1) and must redo its shard;
    every rank must still end with the single-sweep top-m."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist
    from conftest import CASE_SPACE, oracle_ensemble, oracle_space
    from oracle.tuner import top_m
    from paper_1506_00842_b200.distributed import records_protocol, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        osp = oracle_space(CASE_SPACE[case])
        oens = oracle_ensemble(case)
        lo, hi = shard_bounds(osp.card, rank, world)
        calls = {"redo": 0, "gather": 0}

        def record(status):
            i, p = top_m(oens, osp, m, begin=lo, end=hi)
            rec = np.full(2 * m + 1, -1, dtype=np.int64)
            rec[m:2 * m] = np.array([np.inf]).view(np.int64)[0]
            if status == 0:
                rec[:len(i)] = i
                rec[m:m + len(i)] = np.asarray(p, dtype=np.float64).view(np.int64)
            rec[2 * m] = status
            return torch.from_numpy(rec)

        def gather(rec):
            calls["gather"] += 1
            out = torch.empty(world * (2 * m + 1), dtype=torch.int64)
            dist.all_gather_into_tensor(out, rec)
            return out

        def merge(out):
            recs = out.numpy().reshape(world, 2 * m + 1)
            gi = recs[:, :m].reshape(-1)
            gp = recs[:, m:2 * m].reshape(-1).copy().view(np.float64)
            status = int(np.bitwise_or.reduce(recs[:, 2 * m]))
            keep = gi >= 0
            gi, gp = gi[keep], gp[keep]
            o = np.lexsort((gi, gp))[:m]
            return gi[o], gp[o], status

        def redo():
            calls["redo"] += 1
            return record(0)

        i, p = records_protocol(rank, world, m, lambda: record(1 if rank == bad_rank else 0), gather, merge, redo)
        q.put((rank, i.tolist(), p.tolist(), calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bad_rank", [-1, 1])
def test_records_protocol_redoes_overflowed_shards(bad_rank):
    from conftest import golden
    world, m = 2, 200
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_records_worker, args=(r, world, port, "conv_k1", m, bad_rank, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = golden("topm_conv_k1.npz")
    for rank, i, p, calls in res:
        assert i == g["m200_i"].tolist(), rank
        assert p == g["m200_p"].tolist()
        assert calls["gather"] == (1 if bad_rank < 0 else 2)
        assert calls["redo"] == (1 if rank == bad_rank else 0)
