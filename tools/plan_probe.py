"""Host cost of a fresh plan (what every e2e step pays for a new ensemble):
packing the ensemble (Python), mlt_plan_create (C ABI), and the first
mlt_plan_top_m on it (band setup + tables + step) vs a repeat call.
python tools/plan_probe.py [reps]"""
import copy
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1506_00842_b200 import _native as N          # noqa: E402
from paper_1506_00842_b200.model import model_from_json  # noqa: E402
from paper_1506_00842_b200.space import space_from_json  # noqa: E402

G = ROOT / "tests" / "golden"
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
sp = space_from_json(json.loads((G / "spaces.json").read_text())["synthetic-1e8"])
ens = model_from_json(json.loads((G / "model_synth_k16.json").read_text()))
c = N.ctx(0)
ps = N.packed(sp, "space")
oi, op, on, st = np.empty(200, np.int64), np.empty(200), N.C.c_int64(), N.MltSweepStats()
card = sp.cardinality()
rows = []
for r in range(reps + 12):
    e = copy.copy(ens)
    t0 = time.perf_counter()
    pe = N.PackedEnsemble(e)
    t1 = time.perf_counter()
    plan = N.C.c_void_p()
    N.check(N.lib().mlt_plan_create(c, N.C.byref(ps.c), N.C.byref(pe.c), N.C.byref(plan)))
    t2 = time.perf_counter()
    N.check(N.lib().mlt_plan_top_m(plan, 200, 0, card, N.ptr(oi, N.C.c_int64), N.ptr(op, N.C.c_double),
                                   N.C.byref(on), N.C.byref(st)))
    t3 = time.perf_counter()
    N.check(N.lib().mlt_plan_top_m(plan, 200, 0, card, N.ptr(oi, N.C.c_int64), N.ptr(op, N.C.c_double),
                                   N.C.byref(on), N.C.byref(st)))
    t4 = time.perf_counter()
    N.lib().mlt_plan_destroy(plan)
    t5 = time.perf_counter()
    if r >= 12:
        rows.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4))
med = [1e3 * statistics.median(x) for x in zip(*rows)]
print(json.dumps({"pack_ms": med[0], "plan_create_ms": med[1], "first_top_m_ms": med[2], "repeat_top_m_ms": med[3],
                  "destroy_ms": med[4], "fresh_overhead_ms": med[0] + med[1] + med[2] - med[3]}))
