"""Public-API wall time of top_m_predicted with and without exact pruning
(a new plan, i.e. fresh tables, every call): python tools/prune_e2e_probe.py"""
import json, sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1506_00842_b200 import tuner as T
from paper_1506_00842_b200.model import model_from_json
from paper_1506_00842_b200.space import space_from_json
G = ROOT / "tests" / "golden"
sp = space_from_json(json.loads((G / "spaces.json").read_text())["synthetic-1e8"])
ens = model_from_json(json.loads((G / "model_synth_k16.json").read_text()))
if "--once" in sys.argv:   # one pruned call (for an ncu launch list)
    T.set_sweep_pruning(True)
    T.top_m_predicted(ens, sp, 200)
    sys.exit(0)
out = {}
for prune in (False, True):
    T.set_sweep_pruning(prune)
    for _ in range(3):
        T.top_m_predicted(ens, sp, 200)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        res = T.top_m_predicted(ens, sp, 200)
        ts.append(time.perf_counter() - t0)
    out["pruned" if prune else "full"] = {"ms_median": 1e3 * float(np.median(ts)), "ms_min": 1e3 * min(ts),
                                          "top3": [list(c) for c, _ in res[:3]]}
T.set_sweep_pruning(False)
print(json.dumps(out))
