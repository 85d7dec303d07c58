"""Public-API top-m timings on one B200, per call (wall clock, host objects in,
results out): a FRESH ensemble object every call (plan, weights H2D and tables
inside the call) and the cached plan (same ensemble object), on the full
10^8 space and on 1/P slices (one rank's shard at P ranks).

    python tools/e2e_slices.py [calls] > profiles/r02_e2e_slices.jsonl"""
import copy
import gc
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1506_00842_b200 import _native as N          # noqa: E402
from paper_1506_00842_b200 import tuner as T            # noqa: E402
from paper_1506_00842_b200.model import model_from_json  # noqa: E402
from paper_1506_00842_b200.space import space_from_json  # noqa: E402

G = ROOT / "tests" / "golden"
calls = int(sys.argv[1]) if len(sys.argv) > 1 else 30
sp = space_from_json(json.loads((G / "spaces.json").read_text())["synthetic-1e8"])
ens = model_from_json(json.loads((G / "model_synth_k16.json").read_text()))
card = sp.cardinality()
N.ctx(0)


for P in (1, 8):
    hi = card // P
    for mode in ("fresh", "cached"):
        ts = []
        for r in range(calls + 3):
            e = copy.copy(ens) if mode == "fresh" else ens
            t0 = time.perf_counter()
            idx, pred = T.top_m_arrays(e, sp, 200, begin=0, end=hi)
            dt = time.perf_counter() - t0
            if r >= 3:
                ts.append(dt * 1e3)
        print(json.dumps({"slice": P, "configs": hi, "mode": mode, "calls": calls,
                          "ms_median": statistics.median(ts), "ms_min": min(ts), "ms_max": max(ts),
                          "ms_mean": statistics.fmean(ts), "ms_all": [round(t, 3) for t in ts]}), flush=True)
    gc.collect()
