"""Small device workloads for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every kernel family of libmltune_b200.so on a small
golden case, each result checked against the oracle so a case that runs
but computes garbage fails too.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py sweep_band

Cases: sweep_band, sweep_pruned_chunked, band_overflow_exact, sweep_groups,
train, surrogate, conv, stereo, raycast, predict_merge, records. `all` runs them in turn.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import (golden, oracle_ensemble, oracle_of_product_ensemble, oracle_space,  # noqa: E402
                      product_ensemble, product_space, surrogates_doc)
from paper_1506_00842_b200 import _native as N  # noqa: E402


def _opt(key, val):
    N.check(N.lib().mlt_ctx_set_option(N.ctx(0), key, val))


def _reset():
    for k in (N.MLT_OPT_PATH, N.MLT_OPT_GROUP, N.MLT_OPT_CAND_CAP, N.MLT_OPT_PRUNE, N.MLT_OPT_CHUNK):
        N.lib().mlt_ctx_set_option(N.ctx(0), k, -1)


def _check_top(ens_case, space_name, m, lo, hi, **stats_want):
    from oracle.tuner import top_m
    from paper_1506_00842_b200.tuner import top_m_arrays
    idx, pred, st = top_m_arrays(product_ensemble(ens_case), product_space(space_name), m, begin=lo, end=hi,
                                 with_stats=True)
    oi, op = top_m(oracle_ensemble(ens_case), oracle_space(space_name), m, begin=lo, end=hi)
    assert np.array_equal(idx, oi), (ens_case, lo, hi)
    assert np.allclose(pred, op, rtol=1e-12, atol=0)
    for k, v in stats_want.items():
        assert st[k] == v, (k, st[k], v)
    return st


def sweep_band():
    """k_table_outer/inner + k_sweep<3,false> + k_band_filter + k_rescore + k_sort_small."""
    _reset()
    st = _check_top("stereo_k8", "stereo", 50, 0, 1 << 18, path=0)
    return {"group": st["group"], "candidates": st["candidates"]}


def sweep_pruned_chunked():
    """k_sweep<3,true> with the pruning tables, several chunks per slice."""
    _reset()
    _opt(N.MLT_OPT_PRUNE, 1)
    _opt(N.MLT_OPT_CHUNK, 1 << 16)
    st = _check_top("stereo_k8", "stereo", 40, 100_000, 100_000 + (1 << 18), path=0)
    _reset()
    return {"evaluated_frac": st["evaluated_frac"]}


def band_overflow_exact():
    """Candidate-buffer overflow -> exact fp64 path (k_predict64 + CUB sort), and m > 1024."""
    _reset()
    _opt(N.MLT_OPT_CAND_CAP, 64)
    _check_top("conv_k11", "convolution", 100, 0, 1 << 15)
    _reset()
    _check_top("conv_k11", "convolution", 1500, 0, 1 << 15)
    return {}


def sweep_groups():
    """Reciprocal groupings G = 1, 2, 4 of the sweep kernel (k = 11 gives 330
    units, not a multiple of 4: the G = 4 request falls back to 3; the k = 8
    stereo ensemble has 240 units and runs G = 4)."""
    out = {}
    for g in (1, 2, 4):
        _reset()
        _opt(N.MLT_OPT_GROUP, g)
        out[f"g{g}"] = _check_top("raycast_k11", "raycasting", 20, 0, 1 << 17)["group"]
    _reset()
    _opt(N.MLT_OPT_GROUP, 4)
    out["g4_stereo"] = _check_top("stereo_k8", "stereo", 50, 0, 1 << 18)["group"]
    _reset()
    return out


def train():
    """k_train on golden case b (k = 3 members, 60 epochs) vs the oracle trainer."""
    from oracle.model import OTrainCfg, fold_rows, fit
    from paper_1506_00842_b200 import model as M
    g = golden("train_small.npz")
    sp = product_space("bench512")
    cfgv = g["b_cfg"]
    idx, times = g["b_idx"], g["b_time"]
    ok = np.isfinite(times) & (times > 0)
    enc = M.Encoder.from_space(sp)
    X = enc.encode_indices(idx[ok])
    y = np.log(times[ok])
    cfg = M.TrainConfig(epochs=int(cfgv[0]), learning_rate=float(cfgv[1]), batch_size=int(cfgv[2]),
                        momentum=float(cfgv[3]), weight_init_scale=float(cfgv[4]), seed=int(cfgv[5]))
    k = int(cfgv[6])
    rows = fold_rows(X.shape[0], k, cfg.seed)
    nets = M.fit_members(X, y, rows, cfg, [(cfg.seed, i) for i in range(k)])
    ocfg = OTrainCfg(cfg.epochs, cfg.learning_rate, cfg.batch_size, cfg.momentum, cfg.weight_init_scale, cfg.seed)
    for i, (net, r) in enumerate(zip(nets, rows)):
        o = fit(X[r], y[r], ocfg, (cfg.seed, i))
        assert np.allclose(net.weights_hidden, o.W1, rtol=1e-8, atol=1e-10), i
    return {"members": k}


def surrogate():
    """k_surr_times(_masks), k_surr_best(_runs) on the convolution space."""
    from oracle.surrogate import OSurrogate
    from paper_1506_00842_b200.surrogate import B200SurrogateRunner
    name = "convolution"
    doc = surrogates_doc()[name]
    sp = product_space(name)
    r = B200SurrogateRunner(doc, sp)
    o = OSurrogate(doc, oracle_space(name))
    idx = np.arange(0, min(sp.cardinality(), 1 << 14), dtype=np.int64)
    t, ok = r.measured_times(idx, 2)
    ot, ook = o.measured_times(idx, 2)
    assert np.array_equal(ok, ook)
    assert np.allclose(t[ok], ot[ook], rtol=1e-12)
    i, tb, nv, _ = r.exhaustive_best(0, min(sp.cardinality(), 1 << 16), 1)
    return {"best": int(i), "valid": int(nv)}


def conv():
    """k_conv5: TMA tile + register blocking, texture, smem-halo and plain variants."""
    import paper_1506_00842_b200 as b
    from oracle.bench_golden import conv5_box
    from paper_1506_00842_b200.runners import B200ConvRunner
    img = np.random.default_rng(5).random((67, 131), dtype=np.float32)
    r = B200ConvRunner(b.builtin_space("convolution"), width=131, height=67, image=img, default_repetitions=1)
    gold = conv5_box(img)
    n = 0
    for cfg in [(32, 8, 1, 1, 0, 0, 0, 0, 0), (16, 4, 4, 4, 0, 1, 0, 0, 1), (16, 8, 4, 4, 0, 1, 1, 0, 1),
                (8, 8, 2, 2, 1, 0, 0, 1, 0), (32, 4, 1, 2, 0, 1, 0, 1, 0), (64, 4, 4, 4, 0, 1, 0, 0, 1)]:
        _, ok = r.run(cfg, 1)
        if ok:
            assert np.array_equal(r.output(), gold), cfg
            n += 1
    r.close()
    return {"variants": n}


def stereo():
    import paper_1506_00842_b200 as b
    from oracle.bench_golden import stereo_sad
    from paper_1506_00842_b200.runners import B200StereoRunner
    r = B200StereoRunner(b.builtin_space("stereo"), width=97, height=61, disparities=16, radius=4, seed=1,
                         default_repetitions=1)
    left, right = r.input()
    gold = stereo_sad(left, right, 16, 4)
    n = 0
    # (wg_x, wg_y, ppt_x, ppt_y, img_left, img_right, local_left, local_right,
    #  unroll_disparity, unroll_diff_x, unroll_diff_y): global, textures, smem
    # tiles, the packed-row path (both tiles local, diff_x = 4)
    for cfg in [(16, 8, 1, 1, 0, 0, 0, 0, 1, 1, 1), (16, 8, 1, 1, 0, 0, 1, 1, 4, 4, 1), (8, 8, 2, 2, 1, 1, 0, 0, 2, 1, 2),
                (32, 4, 1, 1, 0, 0, 1, 1, 1, 4, 4), (16, 8, 2, 1, 0, 1, 1, 0, 8, 2, 4)]:
        _, ok = r.run(cfg, 1)
        if ok:
            assert np.array_equal(r.output(), gold), cfg
            n += 1
    r.close()
    return {"variants": n}


def raycast():
    import paper_1506_00842_b200 as b
    from oracle.bench_golden import raycast as ray
    from paper_1506_00842_b200.runners import B200RaycastRunner
    r = B200RaycastRunner(b.builtin_space("raycasting"), width=67, height=53, volume_shape=(48, 40, 56), seed=4,
                          default_repetitions=1)
    gold = ray(r.volume(), r.transfer(), r.camera(), 67, 53)
    n = 0
    for cfg in [(16, 8, 1, 1, 0, 0, 0, 0, 0, 1), (16, 8, 1, 1, 1, 1, 1, 0, 1, 4), (8, 8, 2, 2, 0, 0, 0, 1, 0, 8)]:
        _, ok = r.run(cfg, 1)
        if ok:
            assert np.array_equal(r.output(), gold), cfg
            n += 1
    r.close()
    return {"variants": n}


def predict_merge():
    """k_decode, k_valid, k_encode, k_predict64, k_member_out64, mlt_merge_top_m."""
    import torch
    from paper_1506_00842_b200.distributed import _device_merge
    from paper_1506_00842_b200.tuner import top_m_arrays
    sp, ens = product_space("conv-rules"), product_ensemble("conv_k11")
    idx = np.arange(0, 5000, 7, dtype=np.int64)
    sp.decode_indices(idx)
    sp.valid_mask_indices(idx)
    p = ens.predict_indices(idx)
    o = oracle_of_product_ensemble(ens).predict_indices(idx)
    assert np.allclose(p, o, rtol=1e-12)
    ens.members[0].forward_batch(ens.encoder.encode_indices(idx[:10]))
    parts = [top_m_arrays(ens, product_space("convolution"), 30, begin=a, end=a + 16384) for a in (0, 16384)]
    gi = torch.tensor(np.concatenate([q[0] for q in parts]), device="cuda")
    gp = torch.tensor(np.concatenate([q[1] for q in parts]), device="cuda")
    mi, _ = _device_merge(gi, gp, 30)
    whole = top_m_arrays(ens, product_space("convolution"), 30, begin=0, end=32768)
    assert np.array_equal(mi, whole[0])
    del gi, gp
    torch.cuda.empty_cache()   # torch's caching allocator would otherwise show as a leak
    return {}


def records():
    """mlt_plan_top_m_record (the record written by the band stage's sort kernel) for 4 shards
    + mlt_merge_records (k_merge_records: one-CTA rank merge), and a forced
    overflow record."""
    import torch
    from paper_1506_00842_b200.distributed import shard_bounds
    sp, ens = product_space("stereo"), product_ensemble("stereo_k8")
    lo_all, hi_all = 0, 1 << 19
    m, world = 40, 4
    plan = N.plan(sp, ens, 0)
    out = torch.empty((world, 2 * m + 1), dtype=torch.int64, device="cuda:0")
    N.check(N.lib().mlt_ctx_set_stream(N.ctx(0), N.C.c_void_p(N.stream_handle(torch.cuda.current_stream()))))
    for r in range(world):
        lo, hi = shard_bounds(hi_all - lo_all, r, world)
        N.check(N.lib().mlt_plan_top_m_record(plan.h, m, lo, hi, N.C.c_void_p(out[r].data_ptr())))
    oi, op = np.empty(m, np.int64), np.empty(m, np.float64)
    on, ost = N.C.c_int64(0), N.C.c_int64(0)
    N.check(N.lib().mlt_merge_records(N.ctx(0), N.C.c_void_p(out.data_ptr()), world, m, N.ptr(oi, N.C.c_int64),
                                      N.ptr(op, N.C.c_double), N.C.byref(on), N.C.byref(ost)))
    from oracle.tuner import top_m
    ri, rp = top_m(oracle_ensemble("stereo_k8"), oracle_space("stereo"), m, begin=lo_all, end=hi_all)
    assert ost.value == 0 and np.array_equal(oi[:on.value], ri)
    _opt(N.MLT_OPT_CAND_CAP, 8)
    N.check(N.lib().mlt_plan_top_m_record(plan.h, m, 0, 1 << 18, N.C.c_void_p(out[0].data_ptr())))
    _reset()
    assert int(out[0, 2 * m].cpu().numpy()) == 1   # (.item() would leave a torch pinned block behind)
    N.check(N.lib().mlt_ctx_set_stream(N.ctx(0), None))
    del out
    N.clear_plans()
    torch.cuda.empty_cache()
    return {"merged": int(on.value)}


CASES = {f.__name__: f for f in (sweep_band, sweep_pruned_chunked, band_overflow_exact, sweep_groups, train,
                                 surrogate, conv, stereo, raycast, predict_merge, records)}

if __name__ == "__main__":
    names = list(CASES) if sys.argv[1:] in ([], ["all"]) else sys.argv[1:]
    for n in names:
        print(json.dumps({"case": n, "ok": True, **CASES[n]()}), flush=True)
