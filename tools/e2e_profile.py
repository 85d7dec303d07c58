"""Where the public API's fresh-ensemble call spends its host time
(tuner.top_m_predicted with a new ensemble object per call, as bench.py's
e2e leg): cProfile over 40 calls after warm-up, plus the per-call median.
python tools/e2e_profile.py"""
import copy
import cProfile
import json
import pstats
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1506_00842_b200 import _native as N, tuner as T  # noqa: E402
from paper_1506_00842_b200.model import model_from_json     # noqa: E402
from paper_1506_00842_b200.space import space_from_json     # noqa: E402

G = ROOT / "tests" / "golden"
sp = space_from_json(json.loads((G / "spaces.json").read_text())["synthetic-1e8"])
ens = model_from_json(json.loads((G / "model_synth_k16.json").read_text()))
for _ in range(12):
    T.top_m_predicted(copy.copy(ens), sp, 200)
ts = []
for _ in range(20):
    e = copy.copy(ens)
    t0 = time.perf_counter()
    T.top_m_predicted(e, sp, 200)
    ts.append(time.perf_counter() - t0)
print(json.dumps({"fresh_call_ms_median": 1e3 * statistics.median(ts)}))
pr = cProfile.Profile()
es = [copy.copy(ens) for _ in range(40)]
pr.enable()
for e in es:
    T.top_m_predicted(e, sp, 200)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
