"""A12: the surrogate device on the B200 against the reference-pinned oracle
(oracle/surrogate.py, itself checked bit-for-bit against the reference's
stage-1 fixtures by test_oracle_golden.py): noise-free times bit-identical,
noisy times within 1e-13 relative, exhaustive search identical."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, oracle_space, product_space, spaces_doc, surrogates_doc

pytestmark = pytest.mark.gpu

NOISY_RTOL = 1e-13     # normcdfinv / exp vs scipy ndtri / glibc exp: a few ulp

CASES = ["convolution", "raycasting", "stereo", "synthetic-1e8", "bench512"]


def _runners(name, space_name=None):
    from oracle.surrogate import OSurrogate
    from paper_1506_00842_b200 import B200SurrogateRunner
    sn = space_name or name
    doc = surrogates_doc()[name]
    return B200SurrogateRunner(doc, product_space(sn)), OSurrogate(doc, oracle_space(sn))


def _probe(name):
    g = golden(f"probe_{name}.npz")
    return g["idx"]


@pytest.mark.parametrize("name", CASES)
def test_true_times_bit_exact(gpu_ok, name):
    dev, ora = _runners(name)
    idx = _probe(name)
    t, ok = dev.true_times(idx)
    to, oko = ora.true_times(idx)
    assert np.array_equal(ok, oko)
    np.testing.assert_array_equal(t, to)          # NaN where a launch rule fires, else bit-identical
    assert (~ok).any() or name in ("bench512",)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("reps", [1, 3])
def test_measured_times_match(gpu_ok, name, reps):
    dev, ora = _runners(name)
    idx = _probe(name)
    t, ok = dev.measured_times(idx, reps)
    to, oko = ora.measured_times(idx, reps)
    assert np.array_equal(ok, oko)
    np.testing.assert_allclose(t[ok], to[ok], rtol=NOISY_RTOL, atol=0)
    assert np.isnan(t[~ok]).all()


@pytest.mark.parametrize("name", ["convolution", "raycasting", "stereo", "synthetic-1e8"])
def test_stage1_fixture_reproduced(gpu_ok, name):
    """The reference's own stage-1 measurements (tests/golden, made by the real
    SurrogateRunner) through the device runner's measure()."""
    dev, _ = _runners(name)
    g = golden(f"stage1_{name}.npz")
    sp = product_space(name)
    for q in range(0, g["idx"].shape[0], 97):         # the scalar path on a stride
        s = dev.measure(sp.config_at(int(g["idx"][q])))
        assert s.outcome.is_valid == bool(g["ok"][q])
        if s.outcome.is_valid:
            assert s.outcome.time == pytest.approx(float(g["time"][q]), rel=NOISY_RTOL, abs=0)
    t, ok = dev.measured_times(g["idx"], 1)           # and the batch path on all of it
    assert np.array_equal(ok, g["ok"])
    np.testing.assert_allclose(t[ok], g["time"][ok], rtol=NOISY_RTOL, atol=0)


def _oracle_best(ora, card, reps, chunk=1 << 20, thr=np.nan, static=None):
    best, nv, nb = None, 0, 0
    for s in range(0, card, chunk):
        idx = np.arange(s, min(s + chunk, card), dtype=np.int64)
        if static is not None:
            idx = idx[static(idx)]
        t, ok = ora.true_times(idx) if reps == 0 else ora.measured_times(idx, reps)
        if not ok.any():
            continue
        nv += int(ok.sum())
        nb += int((t[ok] < thr).sum())
        tt = np.where(ok, t, np.inf)
        p = int(np.argmin(tt))
        key = (float(tt[p]), int(idx[p]))
        if best is None or key < best:
            best = key
    return best, nv, nb


@pytest.mark.parametrize("name", ["convolution", "raycasting", "stereo"])
@pytest.mark.parametrize("reps", [0, 1, 2])
def test_exhaustive_best_matches_oracle(gpu_ok, name, reps):
    dev, ora = _runners(name)
    card = product_space(name).cardinality()
    (bt, bi), nv, _ = _oracle_best(ora, card, reps)
    thr = bt * 1.5
    i, t, n_valid, n_below = dev.exhaustive_best(repetitions=reps, threshold=thr)
    _, _, nb = _oracle_best(ora, card, reps, thr=thr)
    assert i == bi and n_valid == nv and n_below == nb
    if reps == 0:
        assert t == bt
    else:
        assert t == pytest.approx(bt, rel=NOISY_RTOL, abs=0)


def test_exhaustive_conv_gpu_a_optimum(gpu_ok):
    """the conv gpu-a optimum is index 88599 at 0.014444711 s,
    and exhaustive_search dispatches to the fused device sweep."""
    import paper_1506_00842_b200 as b
    dev, _ = _runners("convolution")
    sp = product_space("convolution")
    cfg, t = b.exhaustive_search(sp, dev)
    assert sp.index_of(cfg) == 88599 and t == pytest.approx(0.014444711, rel=1e-7)


def test_exhaustive_respects_static_rules_and_slices(gpu_ok):
    """conv-rules space (one static rule of every kind) x the conv spec; slices
    of the range agree with the whole."""
    from oracle.surrogate import OSurrogate
    from paper_1506_00842_b200 import B200SurrogateRunner
    doc = surrogates_doc()["convolution"]
    osp = oracle_space("conv-rules")
    ora = OSurrogate(doc, osp)
    dev = B200SurrogateRunner(doc, product_space("conv-rules"))
    card = product_space("conv-rules").cardinality()
    static = lambda idx: osp.rule_mask(osp.rules, osp.decode(idx))   # noqa: E731
    (bt, bi), nv, _ = _oracle_best(ora, card, 1, static=static)
    i, t, n_valid, _ = dev.exhaustive_best()
    assert (i, n_valid) == (bi, nv) and t == pytest.approx(bt, rel=NOISY_RTOL)
    parts = [dev.exhaustive_best(a, min(a + 40000, card)) for a in range(0, card, 40000)]
    assert sum(p[2] for p in parts) == nv
    assert min((p[1], p[0]) for p in parts if p[0] >= 0)[1] == bi
    assert dev.exhaustive_best(5, 5) == (-1, pytest.approx(np.nan, nan_ok=True), 0, 0)


def test_synthetic_1e8_exhaustive_consistent_with_times(gpu_ok):
    """The full 10^8 space in one fused sweep; a 2^21 slice cross-checked
    against the oracle, and the global best re-measured on the oracle."""
    dev, ora = _runners("synthetic-1e8")
    card = product_space("synthetic-1e8").cardinality()
    i, t, n_valid, _ = dev.exhaustive_best()
    assert 0 < n_valid < card and 0 <= i < card
    to, oko = ora.measured_times(np.array([i]), 1)
    assert oko[0] and t == pytest.approx(float(to[0]), rel=NOISY_RTOL)
    lo, hi = 50_000_000, 50_000_000 + (1 << 21)
    idx = np.arange(lo, hi, dtype=np.int64)
    tt, ok = ora.measured_times(idx, 1)
    p = int(np.argmin(np.where(ok, tt, np.inf)))
    j, tj, nvj, _ = dev.exhaustive_best(lo, hi)
    assert j == int(idx[p]) and nvj == int(ok.sum()) and tj == pytest.approx(float(tt[p]), rel=NOISY_RTOL)
    assert t <= tj


def test_spec_errors(gpu_ok):
    from paper_1506_00842_b200 import B200SurrogateRunner, ConfigMismatchError
    sp = product_space("convolution")
    with pytest.raises(ConfigMismatchError):
        B200SurrogateRunner({"base_time": 1.0, "terms": [{"params": ["nope"], "match": [1], "factor": 2.0}]}, sp)
    with pytest.raises(ValueError):
        B200SurrogateRunner({"base_time": 0.0}, sp)
    r = B200SurrogateRunner({"base_time": 2.0, "terms": [{"params": ["wg_x"], "match": [3], "factor": 9.0}]}, sp)
    t, ok = r.true_times(np.arange(10))
    assert ok.all() and (t == 2.0).all()          # a value not in the list never matches
    assert spaces_doc()["convolution"]["name"] == "convolution"


def _sharded_worker(rank, world, port, q):
    import os
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch
    import torch.distributed as dist
    from conftest import product_space, surrogates_doc
    from paper_1506_00842_b200 import B200SurrogateRunner
    from paper_1506_00842_b200.distributed import exhaustive_search

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)                 # functional run: both ranks share the one B200
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sp = product_space("synthetic-1e8")
        r = B200SurrogateRunner(surrogates_doc()["synthetic-1e8"], sp)
        cfg, t = exhaustive_search(sp, r)
        q.put((rank, sp.index_of(cfg), t))
    finally:
        dist.destroy_process_group()


def test_sharded_exhaustive_on_device(gpu_ok):
    """distributed.exhaustive_search over 2 gloo ranks (device search per slice,
    one all-gather) == the single-GPU fused search of the 10^8 space."""
    import socket

    import torch.multiprocessing as mp
    dev, _ = _runners("synthetic-1e8")
    i1, t1, _, _ = dev.exhaustive_best()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, i, t in res:
        assert i == i1 and t == t1, rank
