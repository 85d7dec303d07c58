"""BASELINE configs[4]: the end-to-end auto-tuning loop on the B200 convolution
benchmark (4096 x 4096 fp32, 5x5 box filter) versus exhaustive search.

    python tools/conv_autotune.py --sample 300            # time distribution of random configs
    python tools/conv_autotune.py --tune --exhaustive     # the full experiment

Every measurement is the B200 kernel itself (CUDA events, min over
repetitions, L2 flushed before each run). Prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1506_00842_b200 as b  # noqa: E402
from paper_1506_00842_b200.runners import B200ConvRunner  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--sample", type=int, default=0)
    ap.add_argument("--tune", action="store_true")
    ap.add_argument("--exhaustive", action="store_true")
    ap.add_argument("--n-train", type=int, default=2000)
    ap.add_argument("--m", type=int, nargs="+", default=[10, 200])
    ap.add_argument("--seeds", type=int, nargs="+", default=[0])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--budget-s", type=float, default=1800.0, help="stop the exhaustive sweep after this long")
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    space = b.builtin_space("convolution")
    runner = B200ConvRunner(space, width=args.size, height=args.size, seed=0, default_repetitions=args.reps)
    res = {"experiment": "configs[4]: autotune vs exhaustive, B200 convolution", "image": [args.size, args.size],
           "space": space.name, "cardinality": space.cardinality()}

    if args.sample:
        rng = np.random.default_rng(1)
        idx = rng.choice(space.cardinality(), args.sample, replace=False)
        t0 = time.perf_counter()
        times, ok = runner.measured_times(idx, 1)
        res["sample"] = {"n": int(args.sample), "valid": int(ok.sum()), "wall_s": time.perf_counter() - t0,
                         "ms_quantiles": {q: float(np.nanquantile(times[ok], q) * 1e3) for q in (0, 0.1, 0.5, 0.9, 0.99, 1)},
                         "ms_mean": float(np.nanmean(times[ok]) * 1e3)}

    if args.tune:
        res["tune"] = []
        for seed in args.seeds:
            for m in args.m:
                t0 = time.perf_counter()
                rep = b.autotune(space, runner, b.TunerConfig(n_train=args.n_train, m_candidates=m, k_bag=11, seed=seed))
                res["tune"].append({"seed": seed, "m": m, "best_index": rep.best_index, "best_config": rep.best_config,
                                    "best_time_s": rep.best_time, "predicted_best_s": rep.predicted_best_time,
                                    "stage2_invalid": rep.stage2_invalid_count, "wall_s": time.perf_counter() - t0})

    if args.exhaustive:
        card = space.cardinality()
        t0 = time.perf_counter()
        times = np.full(card, np.nan)
        done = 0
        for s in range(0, card, 4096):
            idx = np.arange(s, min(s + 4096, card))
            t, ok = runner.measured_times(idx, 1)
            times[idx[ok]] = t[ok]
            done = idx[-1] + 1
            if time.perf_counter() - t0 > args.budget_s:
                break
        wall = time.perf_counter() - t0
        order = np.argsort(np.where(np.isnan(times), np.inf, times))[:20]
        # re-measure the 20 fastest with the tuner's repetitions
        best = None
        for i in order.tolist():
            tt, ok = runner.run(space.config_at(i), args.reps)
            if ok and (best is None or (tt, i) < best):
                best = (tt, i)
        res["exhaustive"] = {"measured": int(done), "complete": bool(done == card), "valid": int(np.isfinite(times).sum()),
                             "wall_s": wall, "best_index": best[1], "best_config": space.config_at(best[1]),
                             "best_time_s": best[0]}
        for t in res.get("tune", []):
            t["slowdown_vs_exhaustive"] = t["best_time_s"] / best[0]
    runner.close()
    line = json.dumps(res)
    print(line)
    if args.out:
        Path(args.out).write_text(line + "\n")


if __name__ == "__main__":
    main()
