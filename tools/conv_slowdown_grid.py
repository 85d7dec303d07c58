"""The paper's tuning-quality experiment on real hardware: mean slowdown of the
auto-tuner's pick vs the exhaustive optimum over an (N, M) grid
(evaluation.slowdown_grid) with the B200 4096^2 convolution
kernel as the device under tuning. One repetition per measurement (CUDA
events, L2 flushed). Prints one JSON line.

    python tools/conv_slowdown_grid.py [--n 500 1000 2000] [--m 10 50 200] [--repeats 3]
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1506_00842_b200 as b  # noqa: E402
from paper_1506_00842_b200 import evaluation as EV  # noqa: E402
from paper_1506_00842_b200.runners import B200ConvRunner  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[500, 1000, 2000])
    ap.add_argument("--m", type=int, nargs="+", default=[10, 50, 200])
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    space = b.builtin_space("convolution")
    runner = B200ConvRunner(space, a.size, a.size, default_repetitions=1)
    t0 = time.perf_counter()
    cfg, opt = b.exhaustive_search(space, runner)
    ex_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    cells = EV.slowdown_grid(space, runner, a.n, a.m, a.repeats, 2015, k=11)
    grid_s = time.perf_counter() - t0
    res = {"experiment": "slowdown grid, B200 convolution 4096^2 (paper's tuning-quality experiment)",
           "exhaustive": {"best_config": list(cfg), "best_time_s": opt, "wall_s": ex_s},
           "grid_wall_s": grid_s, "repetitions": 1,
           "cells": [{"n": c.n_train, "m": c.m_candidates, "mean_slowdown": c.mean_slowdown, "n_success": c.n_success,
                      "n_invalid_runs": c.invalid_run_count} for c in cells]}
    runner.close()
    line = json.dumps(res)
    print(line)
    if a.out:
        Path(a.out).write_text(line + "\n")


if __name__ == "__main__":
    main()
