"""The device-resident sharded step: `mlt_plan_top_m_record`
writes each shard's top-m into a device record with no host round trip and
`mlt_merge_records` merges the gathered records on the device. On one B200
the P shards of a P-GPU run are swept in turn into one buffer (what the NCCL
all-gather would assemble); the merge must equal the reference's golden top-m
of the whole space, and a forced guard-band overflow must surface as a
status word (the protocol then redoes that shard exactly)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import CASE_SPACE, golden, product_ensemble, product_space

pytestmark = pytest.mark.gpu


def _records(ens, sp, m, world, torch, begin=0, end=None):
    from paper_1506_00842_b200 import _native as N
    from paper_1506_00842_b200.distributed import shard_bounds
    plan = N.plan(sp, ens, 0)
    card = sp.cardinality() if end is None else end
    out = torch.full((world, 2 * m + 1), 7, dtype=torch.int64, device="cuda:0")
    # on torch's stream, so torch reads of `out` are ordered behind the records
    with N.on_stream(0, torch.cuda.current_stream().cuda_stream):
        for r in range(world):
            lo, hi = shard_bounds(card - begin, r, world)
            N.check(N.lib().mlt_plan_top_m_record(plan.h, m, begin + lo, begin + hi,
                                                  N.C.c_void_p(out[r].data_ptr())))
    return out


def _merge(out, world, m):
    from paper_1506_00842_b200 import _native as N
    oi, op = np.empty(m, np.int64), np.empty(m, np.float64)
    on, ost = N.C.c_int64(0), N.C.c_int64(0)
    N.check(N.lib().mlt_merge_records(N.ctx(0), N.C.c_void_p(out.data_ptr()), world, m, N.ptr(oi, N.C.c_int64),
                                      N.ptr(op, N.C.c_double), N.C.byref(on), N.C.byref(ost)))
    return oi[:on.value], op[:on.value], ost.value


@pytest.mark.parametrize("case", ["conv_k11", "stereo_k8", "synth_k16"])
@pytest.mark.parametrize("world", [1, 2, 8])
def test_records_merge_equals_golden(gpu_ok, case, world):
    import torch
    sp, ens = product_space(CASE_SPACE[case]), product_ensemble(case)
    g = golden(f"topm_{case}.npz")
    for m in (10, 200):
        if f"m{m}_i" not in g:
            continue
        out = _records(ens, sp, m, world, torch)
        idx, pred, status = _merge(out, world, m)
        assert status == 0
        assert np.array_equal(idx, g[f"m{m}_i"]), (case, world, m)
        np.testing.assert_allclose(pred, g[f"m{m}_p"], rtol=1e-12, atol=0)


def test_records_padding_small_shards_and_exact_path(gpu_ok):
    """Shards with fewer than m valid configurations pad with (-1, +inf);
    m > 1024 takes the exact path inside the record call; both merge exactly."""
    import torch
    from paper_1506_00842_b200.tuner import top_m_arrays
    sp, ens = product_space("convolution"), product_ensemble("conv_k11")
    for lo, hi, m, world in [(100, 140, 50, 4), (0, 1 << 16, 1500, 3), (5000, 5003, 7, 2)]:
        out = _records(ens, sp, m, world, torch, begin=lo, end=hi)
        idx, pred, status = _merge(out, world, m)
        ref = top_m_arrays(ens, sp, m, begin=lo, end=hi)
        assert status == 0
        assert np.array_equal(idx, ref[0]) and np.array_equal(pred, ref[1]), (lo, hi, m)


def test_records_report_overflow(gpu_ok):
    """A candidate buffer too small for the band: the record says so (status 1)
    instead of returning a wrong list."""
    import torch
    from paper_1506_00842_b200 import _native as N
    sp, ens = product_space("stereo"), product_ensemble("stereo_k8")
    N.check(N.lib().mlt_ctx_set_option(N.ctx(0), N.MLT_OPT_CAND_CAP, 16))
    try:
        out = _records(ens, sp, 100, 2, torch)
    finally:
        N.lib().mlt_ctx_set_option(N.ctx(0), N.MLT_OPT_CAND_CAP, -1)
    st = out[:, 200].cpu().numpy()
    assert (st == 1).all(), st
    _, _, status = _merge(out, 2, 100)
    assert status == 1


def test_records_protocol_single_rank_gloo(gpu_ok):
    """top_m_arrays_records end to end in a one-rank gloo group (the collective
    runs on host tensors; the sweep and the merge on the device)."""
    import os
    import socket

    import torch.distributed as dist
    from paper_1506_00842_b200.distributed import top_m_arrays_records
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        sp, ens = product_space("stereo"), product_ensemble("stereo_k8")
        g = golden("topm_stereo_k8.npz")
        idx, pred = top_m_arrays_records(ens, sp, 200)
        assert np.array_equal(idx, g["m200_i"])
    finally:
        dist.destroy_process_group()


def test_records_merge_ties_and_large_merges(gpu_ok):
    """The rank merge orders equal predictions by index across records (a
    constant ensemble: every configuration ties, the answer is the first m
    valid indices); a merge beyond the one-CTA capacity (n_rec * m > 8192)
    takes the sort path; both equal the single-call top-m."""
    import torch
    from paper_1506_00842_b200.model import Encoder, Ensemble, Network
    from paper_1506_00842_b200.tuner import top_m_arrays
    sp = product_space("stereo")
    rng = np.random.default_rng(3)
    d = len(sp.params)
    flat = Ensemble([Network(np.zeros((30, d)), rng.uniform(-1, 1, 30), rng.uniform(-1, 1, 30), 0.2, 1.0, 1.5)
                     for _ in range(4)], Encoder.from_space(sp), sp.name)
    for world, m in [(4, 300), (8, 100), (3, 1000)]:
        out = _records(flat, sp, m, world, torch)
        idx, pred, status = _merge(out, world, m)
        ref = top_m_arrays(flat, sp, m)
        assert status == 0
        assert np.array_equal(idx, ref[0]) and np.array_equal(pred, ref[1]), (world, m)
    ens = product_ensemble("stereo_k8")
    for world, m in [(3, 3000), (2, 4096)]:
        out = _records(ens, sp, m, world, torch)
        idx, pred, status = _merge(out, world, m)
        ref = top_m_arrays(ens, sp, m)
        assert status == 0
        assert np.array_equal(idx, ref[0]), (world, m)
        np.testing.assert_allclose(pred, ref[1], rtol=1e-12, atol=0)
