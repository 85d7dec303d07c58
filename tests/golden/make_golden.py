"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Runs only in the build container, where the reference package `mltune` is
importable read-only from /root/reference/pkg/src. Nothing on the GPU box
runs this; the tests there read the committed fixtures it wrote.

    python tests/golden/make_golden.py            # everything except the 1e8 sweep
    python tests/golden/make_golden.py --synth    # also the full 1e8 reference sweep (~8 min)

Fixtures (all small):
  spaces.json        space JSON per case (reference space_to_json)
  surrogates.json    surrogate spec JSON per case (reference surrogate_to_json)
  stage1_<case>.npz  stage-1 sample set: idx, ok, time (reference autotune stage 1)
  model_<case>.json  reference-trained ensemble (reference save_model, 17g floats)
  probe_<space>.npz  seeded probe indices + reference decode / mask / encode
  pred_<case>.npz    probe indices + reference predict_indices
  topm_<case>.npz    reference top_m_predicted (indices, predictions) per m
  train_small.npz    reference _fit outputs on small cases (weights + losses)
  formats/           (--formats) files written by the reference's own writers:
                     sample CSVs, a surrogate spec JSON, a `mltune predict` CSV
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import mltune  # noqa: E402
from mltune import measurement as M  # noqa: E402
from mltune import model as MD  # noqa: E402
from mltune import paramspace as PS  # noqa: E402
from mltune import tuner as T  # noqa: E402
from mltune.profiles import builtin_surrogate  # noqa: E402
from mltune.rng import make_rng  # noqa: E402

OUT = Path(__file__).resolve().parent


def synthetic_space() -> PS.ParamSpace:
    """conv's 9 params + 4 of {1,2,4,8} + 1 of {1,2,3}
    = 131072 * 256 * 3 = 100,663,296 configurations, d = 14."""
    conv = PS.builtin_space("convolution")
    extra = [PS.ParamDef("tile_x", (1, 2, 4, 8)), PS.ParamDef("tile_y", (1, 2, 4, 8)),
             PS.ParamDef("vector", (1, 2, 4, 8)), PS.ParamDef("stages", (1, 2, 4, 8)),
             PS.ParamDef("split", (1, 2, 3))]
    return PS.ParamSpace("synthetic-1e8", conv.params + tuple(extra))


def synthetic_surrogate(space) -> M.SurrogateSpec:
    """gpu-a terms for the conv params plus seeded factors on the 5 new ones."""
    base = builtin_surrogate("gpu-a", space)
    rng = make_rng(1506, 842)
    terms = list(base.terms)
    for p in space.params[9:]:
        for v in p.values[1:]:
            terms.append(M.SurrogateTerm((p.name,), (v,), float(np.exp(rng.uniform(-0.3, 0.3)))))
    terms.append(M.SurrogateTerm(("tile_x", "wg_x"), (8, 128), 1.7))
    terms.append(M.SurrogateTerm(("vector", "ppt_x"), (8, 1), 1.3))
    terms.append(M.SurrogateTerm(("stages", "use_local"), (4, 1), 0.9))
    return M.SurrogateSpec(base_time=base.base_time, terms=tuple(terms),
                           noise_cv=base.noise_cv, invalid_rules=base.invalid_rules,
                           seed=base.seed)


def rules_space() -> PS.ParamSpace:
    """Reduced conv with one rule of every kind, including an int64-wrapping
    product, to pin the mask semantics (paramspace.py:92-107)."""
    conv = PS.builtin_space("convolution")
    rules = (PS.ValidityRule("max-product", ("wg_x", "wg_y"), bound=256),
             PS.ValidityRule("max-weighted-sum", ("ppt_x", "ppt_y", "unroll"), (1, 2, -64), bound=96),
             PS.ValidityRule("forbidden-combination", ("use_image", "use_local", "padding"), (1, 0, 1)),
             PS.ValidityRule("max-product", ("wg_x", "ppt_x", "ppt_y"), (1 << 40, 1 << 20, 3), bound=1 << 50))
    return PS.ParamSpace("conv-rules", conv.params, rules)


def stage1(space, spec, n=2000, seed=0):
    runner = M.SurrogateRunner(spec, space, runner_id="golden")
    configs = space.sample_random(n, seed)
    samples = T.measure_configs(space, runner, configs)
    ss = M.SampleSet(space, "golden", tuple(samples))
    idx = np.array([space.index_of(s.config) for s in samples], dtype=np.int64)
    ok = np.array([s.outcome.is_valid for s in samples])
    tm = np.array([s.outcome.time if s.outcome.is_valid else np.nan for s in samples])
    return ss, idx, ok, tm


def probe_indices(card, n=2048, seed=7):
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, card, size=n - 4, dtype=np.int64)
    return np.concatenate([idx, [0, 1, card - 2, card - 1]]).astype(np.int64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--synth", action="store_true", help="run the full 1e8 reference sweep")
    ap.add_argument("--formats", action="store_true", help="only (re)write the on-disk format fixtures")
    ap.add_argument("--eval", action="store_true", help="only (re)write the evaluation-harness fixture")
    args = ap.parse_args()
    if args.formats:
        return formats_fixtures()
    if args.eval:
        return eval_fixtures()
    t0 = time.time()
    spaces = {n: PS.builtin_space(n) for n in PS.BUILTIN_SPACE_NAMES}
    spaces["synthetic-1e8"] = synthetic_space()
    spaces["conv-rules"] = rules_space()
    import conftest_ref  # noqa: F401  (reference test fixtures, see below)
    spaces["bench512"] = conftest_ref.make_space512()
    spaces["tiny"] = PS.ParamSpace("tiny", (PS.ParamDef("a", (1, 2, 4)), PS.ParamDef("b", (0, 1)),
                                            PS.ParamDef("c", (10, 20, 30, 40))))
    (OUT / "spaces.json").write_text(json.dumps({k: PS.space_to_json(v) for k, v in spaces.items()}, indent=1))

    specs = {
        "convolution": builtin_surrogate("gpu-a", spaces["convolution"]),
        "raycasting": builtin_surrogate("gpu-a", spaces["raycasting"]),
        "stereo": builtin_surrogate("gpu-a", spaces["stereo"]),
        "synthetic-1e8": synthetic_surrogate(spaces["synthetic-1e8"]),
        "bench512": conftest_ref.make_surrogate512(),
    }
    (OUT / "surrogates.json").write_text(json.dumps({k: M.surrogate_to_json(v) for k, v in specs.items()}, indent=1))

    # decode / mask / encode probes (A1-A3)
    for name, sp in spaces.items():
        card = sp.cardinality()
        idx = probe_indices(card) if card > 4096 else np.arange(card, dtype=np.int64)
        vals = sp.decode_indices(idx)
        np.savez_compressed(OUT / f"probe_{name}.npz", idx=idx, values=vals,
                            mask=sp.static_valid_mask(vals),
                            feat=MD.Encoder.from_space(sp).encode_indices(idx))
    print("probes", time.time() - t0, flush=True)

    cases = {  # case -> (space, k, m list)
        "conv_k1": ("convolution", 1, [10, 200]),
        "conv_k11": ("convolution", 11, [1, 10, 200, 1000]),
        "raycast_k11": ("raycasting", 11, [10, 200]),
        "stereo_k8": ("stereo", 8, [10, 200]),
        "synth_k16": ("synthetic-1e8", 16, [200]),
        "b512_k3": ("bench512", 3, [1, 7, 512, 600]),
    }
    stage_cache = {}
    for case, (sname, k, ms) in cases.items():
        sp = spaces[sname]
        if sname not in stage_cache:
            n = 200 if sname == "bench512" else 2000
            stage_cache[sname] = stage1(sp, specs[sname], n=n, seed=0)
            ss, idx, ok, tm = stage_cache[sname]
            np.savez_compressed(OUT / f"stage1_{sname}.npz", idx=idx, ok=ok, time=tm)
        ss = stage_cache[sname][0]
        cfg = MD.TrainConfig(seed=0, epochs=60) if sname == "bench512" else MD.TrainConfig(seed=0)
        ens = MD.train_ensemble(ss, sp, k=k, cfg=cfg, jobs=8)
        MD.save_model(ens, OUT / f"model_{case}.json")
        card = sp.cardinality()
        pidx = probe_indices(card, 4096, seed=11) if card > 4096 else np.arange(card, dtype=np.int64)
        np.savez_compressed(OUT / f"pred_{case}.npz", idx=pidx, pred=ens.predict_indices(pidx),
                            first_loss=np.array([m.first_epoch_loss for m in ens.members]),
                            final_loss=np.array([m.final_epoch_loss for m in ens.members]))
        tops = {}
        if sname == "synthetic-1e8":
            # bounded slices always; the full-space sweep only with --synth
            for lo, hi in ((0, 1 << 21), (card - (1 << 21), card), (37_000_000, 37_000_000 + (1 << 21))):
                sub_idx, sub_pred = slice_top(ens, sp, 200, lo, hi)
                tops[f"slice_{lo}_{hi}_i"] = sub_idx
                tops[f"slice_{lo}_{hi}_p"] = sub_pred
            if args.synth:
                ts = time.time()
                res = T.top_m_predicted(ens, sp, 200)
                tops["m200_i"] = np.array([sp.index_of(c) for c, _ in res], dtype=np.int64)
                tops["m200_p"] = np.array([p for _, p in res])
                tops["full_seconds"] = np.array(time.time() - ts)
        else:
            for m in ms:
                res = T.top_m_predicted(ens, sp, m)
                tops[f"m{m}_i"] = np.array([sp.index_of(c) for c, _ in res], dtype=np.int64)
                tops[f"m{m}_p"] = np.array([p for _, p in res])
            if card > 100_000:   # seeded sweep_cap path (tuner.py:104-105)
                res = T.top_m_predicted(ens, sp, 10, sweep_cap=50_000, seed=3)
                tops["cap_i"] = np.array([sp.index_of(c) for c, _ in res], dtype=np.int64)
                tops["cap_p"] = np.array([p for _, p in res])
        np.savez_compressed(OUT / f"topm_{case}.npz", **tops)
        print(case, time.time() - t0, flush=True)

    # conv-rules: top-m with every rule kind active (reuses the conv ensemble)
    ens = MD.load_model(OUT / "model_conv_k11.json")
    ens = MD.Ensemble(list(ens.members), ens.encoder, "conv-rules")
    tops = {}
    for m in (10, 200):
        res = T.top_m_predicted(ens, spaces["conv-rules"], m)
        tops[f"m{m}_i"] = np.array([spaces["conv-rules"].index_of(c) for c, _ in res], dtype=np.int64)
        tops[f"m{m}_p"] = np.array([p for _, p in res])
    np.savez_compressed(OUT / "topm_conv-rules_k11.npz", **tops)

    # small training cases: full weights pinned (A9-A10)
    small = {}
    sp512 = spaces["bench512"]
    for tag, (n, cfg, k) in {
        "a": (200, MD.TrainConfig(seed=9, epochs=40), 1),
        "b": (100, MD.TrainConfig(seed=5, epochs=60), 3),
        "c": (333, MD.TrainConfig(seed=2, epochs=25, batch_size=7, momentum=0.5, learning_rate=0.05, weight_init_scale=0.7), 4),
        "d": (64, MD.TrainConfig(seed=4, epochs=30, batch_size=1000), 2),
    }.items():
        runner = M.SurrogateRunner(conftest_ref.make_surrogate512(noise_cv=0.05), sp512)
        configs = sp512.sample_random(n, 6)
        ss = M.SampleSet(sp512, "r", tuple(T.measure_configs(sp512, runner, configs)))
        ens = MD.train_ensemble(ss, sp512, k=k, cfg=cfg)
        small[f"{tag}_idx"] = np.array([sp512.index_of(s.config) for s in ss.samples], dtype=np.int64)
        small[f"{tag}_time"] = np.array([s.outcome.time for s in ss.samples])
        small[f"{tag}_cfg"] = np.array([cfg.epochs, cfg.learning_rate, cfg.batch_size, cfg.momentum,
                                        cfg.weight_init_scale, cfg.seed, k], dtype=np.float64)
        for i, mem in enumerate(ens.members):
            small[f"{tag}_{i}_W1"] = mem.weights_hidden
            small[f"{tag}_{i}_b1"] = mem.biases_hidden
            small[f"{tag}_{i}_w2"] = mem.weights_out
            small[f"{tag}_{i}_misc"] = np.array([mem.bias_out, mem.target_mean, mem.target_std,
                                                 mem.first_epoch_loss, mem.final_epoch_loss])
    # divergence case (test_model.py:267-271)
    runner = M.SurrogateRunner(conftest_ref.make_surrogate512(), sp512)
    ss = M.SampleSet(sp512, "r", tuple(T.measure_configs(sp512, runner, sp512.sample_random(60, 6))))
    try:
        MD.train_network(ss, sp512, MD.TrainConfig(seed=1, learning_rate=1e9, momentum=0.0))
        small["div_epoch"] = np.array(-1)
    except mltune.DivergenceError as e:
        small["div_epoch"] = np.array(e.epoch)
    small["div_idx"] = np.array([sp512.index_of(s.config) for s in ss.samples], dtype=np.int64)
    small["div_time"] = np.array([s.outcome.time for s in ss.samples])
    np.savez_compressed(OUT / "train_small.npz", **small)
    print("done", time.time() - t0)


def formats_fixtures():
    """Sample CSV / surrogate JSON / prediction CSV written by the reference's
    own writers (measurement.py:353-554, cli.py:330-353)."""
    from mltune import cli
    d = OUT / "formats"
    d.mkdir(exist_ok=True)
    conv = PS.builtin_space("convolution")
    spec = builtin_surrogate("gpu-a", conv)
    runner = M.SurrogateRunner(spec, conv, runner_id="gpu-a", default_repetitions=2)
    ss = M.SampleSet(conv, "gpu-a", tuple(T.measure_configs(conv, runner, conv.sample_random(300, 4), 2)))
    M.save_samples(ss, d / "samples_convolution.csv")
    M.save_surrogate_spec(spec, d / "surrogate_gpu-a_convolution.json")
    tiny = PS.ParamSpace("tiny", (PS.ParamDef("a", (1, 2, 4)), PS.ParamDef("b", (0, 1)),
                                  PS.ParamDef("c", (10, 20, 30, 40))),
                         (PS.ValidityRule("max-product", ("a", "c"), bound=80),))
    tspec = M.SurrogateSpec(0.5, (M.SurrogateTerm(("a",), (4,), 2.5), M.SurrogateTerm(("b", "c"), (1, 30), 0.4)),
                            noise_cv=0.1, seed=7)
    tr = M.SurrogateRunner(tspec, tiny, runner_id="tiny-sur")
    tss = M.SampleSet(tiny, "tiny-sur", tuple(T.measure_configs(tiny, tr, [tiny.config_at(i) for i in range(24)])))
    M.save_samples(tss, d / "samples_tiny.csv")
    ens = MD.train_ensemble(tss, tiny, k=3, cfg=MD.TrainConfig(seed=3, epochs=50))
    MD.save_model(ens, d / "model_tiny.json")
    assert cli.main(["predict", "--model", str(d / "model_tiny.json"), "--out", str(d / "pred_tiny.csv")]) == 0
    assert cli.main(["predict", "--model", str(OUT / "model_conv_k11.json"), "--index", "4242",
                     "--out", str(d / "pred_conv_4242.csv")]) == 0
    print("formats written to", d)


def eval_fixtures():
    """The reference's learning_curve / slowdown_grid / random_baseline on the
    512-configuration test space (evaluation.py:110-251), default training."""
    import conftest_ref
    from mltune import evaluation as EV
    sp = conftest_ref.make_space512()
    spec = conftest_ref.make_surrogate512(noise_cv=0.05)
    runner = M.SurrogateRunner(spec, sp, runner_id="s512")
    t0 = time.time()
    pts = EV.learning_curve(sp, runner, [40, 80, 160], repeats=2, seed=5, k=3, holdout_size=100)
    cells = EV.slowdown_grid(sp, runner, [60, 120], [4, 16], repeats=2, seed=9, k=3)
    rb = EV.random_baseline(sp, runner, 50, 3)
    doc = {"learning_curve": [{"n_train": p.n_train, "mre": p.mre, "repeat_mres": list(p.repeat_mres),
                               "failure_reasons": list(p.failure_reasons)} for p in pts],
           "slowdown_grid": [{"n_train": c.n_train, "m_candidates": c.m_candidates, "mean_slowdown": c.mean_slowdown,
                              "n_repeats": c.n_repeats, "invalid_run_count": c.invalid_run_count} for c in cells],
           "random_baseline": {"config": list(rb[0]), "time": rb[1]},
           "surrogate": M.surrogate_to_json(spec),
           "args": {"learning_curve": [[40, 80, 160], 2, 5, 3, 100], "slowdown_grid": [[60, 120], [4, 16], 2, 9, 3],
                    "random_baseline": [50, 3], "noise_cv": 0.05}}
    (OUT / "eval_bench512.json").write_text(json.dumps(doc, indent=1))
    print("eval fixtures", time.time() - t0)


def slice_top(ens, sp, m, lo, hi):
    """Reference arithmetic on a contiguous slice: predict_indices over chunks of
    the same size as tuner._SWEEP_CHUNK, then the same lexsort (tuner.py:112-131)."""
    keep_i, keep_p = [], []
    for s in range(lo, hi, T._SWEEP_CHUNK):
        idx = np.arange(s, min(s + T._SWEEP_CHUNK, hi), dtype=np.int64)
        idx = idx[sp.static_valid_mask(sp.decode_indices(idx))]
        keep_i.append(idx)
        keep_p.append(ens.predict_indices(idx))
    idx = np.concatenate(keep_i)
    pred = np.concatenate(keep_p)
    o = np.lexsort((idx, pred))[:m]
    return idx[o], pred[o]


if __name__ == "__main__":
    sys.path.insert(0, str(OUT))
    main()
