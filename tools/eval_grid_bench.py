"""Evaluation-harness throughput: the paper's slowdown
grid on the convolution space with the gpu-a surrogate, batched (one device
training launch for every run of the grid) vs the same runs one autotune at a
time on the device, vs the reference's CPU trainer per member (oracle port,
timed on one member and scaled). Prints one JSON line.

    python tools/eval_grid_bench.py [--repeats 3]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
G = ROOT / "tests" / "golden"

import paper_1506_00842_b200 as b  # noqa: E402
from paper_1506_00842_b200 import evaluation as EV  # noqa: E402
from paper_1506_00842_b200.space import derive_seed, space_from_json  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--n", type=int, nargs="+", default=[500, 1000, 2000])
    ap.add_argument("--m", type=int, nargs="+", default=[10, 50, 200])
    ap.add_argument("--k", type=int, default=11)
    ap.add_argument("--cpu-member", action="store_true", help="time one member of the reference CPU trainer")
    ap.add_argument("--space", default="convolution", choices=["convolution", "raycasting", "stereo", "synthetic-1e8"])
    ap.add_argument("--no-sequential", action="store_true", help="skip the one-autotune-at-a-time comparison")
    a = ap.parse_args()
    sp = space_from_json(json.loads((G / "spaces.json").read_text())[a.space])
    runner = b.B200SurrogateRunner(json.loads((G / "surrogates.json").read_text())[a.space], sp,
                                   runner_id="gpu-a")
    EV.slowdown_grid(sp, runner, [200], [10], 1, 99, k=3, train_cfg=b.TrainConfig(epochs=5))   # warm-up
    t0 = time.perf_counter()
    cells = EV.slowdown_grid(sp, runner, a.n, a.m, a.repeats, 7, k=a.k)
    batched = time.perf_counter() - t0
    runs = len(a.n) * len(a.m) * a.repeats
    out = {"experiment": f"slowdown_grid, {a.space} space, device surrogate (golden spec)",
           "grid": {"n": a.n, "m": a.m, "repeats": a.repeats, "k": a.k, "runs": runs, "members": runs * a.k},
           "batched_wall_s": batched,
           "cells": [{"n": c.n_train, "m": c.m_candidates, "mean_slowdown": c.mean_slowdown} for c in cells]}
    if not a.no_sequential:
        # the same runs, one autotune call after another (device path, unbatched)
        t0 = time.perf_counter()
        seq_slow = {}
        _, opt = b.exhaustive_search(sp, runner)
        for ci, n in enumerate(a.n):
            for cj, m in enumerate(a.m):
                cid = ci * len(a.m) + cj
                for rep in range(a.repeats):
                    r = b.autotune(sp, runner, b.TunerConfig(n_train=n, m_candidates=m, k_bag=a.k,
                                                             seed=derive_seed(7, cid, rep)))
                    seq_slow.setdefault(cid, []).append(r.best_time / opt)
        out["sequential_device_wall_s"] = time.perf_counter() - t0
        out["identical_results"] = all(abs(c.mean_slowdown - float(np.mean(seq_slow[i]))) <= 1e-12 * c.mean_slowdown
                                       for i, c in enumerate(cells))
    if a.cpu_member:
        from oracle.model import OTrainCfg, fit
        from oracle.space import space_from_doc
        osp = space_from_doc(json.loads((G / "spaces.json").read_text())["convolution"])
        st = np.load(G / "stage1_convolution.npz")
        X = osp.encode(st["idx"][st["ok"]])
        y = np.log(st["time"][st["ok"]])
        t0 = time.perf_counter()
        fit(X, y, OTrainCfg(seed=0), (0, 0))
        per = time.perf_counter() - t0
        mean_n = float(np.mean(a.n)) / 2000.0
        out["cpu_reference_member_s_at_n2000"] = per
        out["cpu_reference_grid_training_s_estimate"] = per * mean_n * runs * a.k * (a.k - 1) / a.k
    print(json.dumps(out))


if __name__ == "__main__":
    main()
