"""A/B timing of sweep-kernel builds: MLTUNE_B200_LIB=<so> python tools/sweep_ab.py [workload] [reps]
Prints one JSON line: sweep kernel ms (CUDA events inside the library), step ms, parity."""
import json, os, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1506_00842_b200 import _native as N
from paper_1506_00842_b200.model import model_from_json
from paper_1506_00842_b200.space import space_from_json

G = ROOT / "tests" / "golden"
case = {"synthetic-1e8": "synth_k16", "stereo": "stereo_k8"}[sys.argv[1] if len(sys.argv) > 1 else "synthetic-1e8"]
name = "synthetic-1e8" if case == "synth_k16" else "stereo"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
sp = space_from_json(json.loads((G / "spaces.json").read_text())[name])
ens = model_from_json(json.loads((G / f"model_{case}.json").read_text()))
c = N.ctx(0)
N.check(N.lib().mlt_ctx_set_profiling(c, 1))
if os.environ.get("MLT_GROUP"):
    N.check(N.lib().mlt_ctx_set_option(c, N.MLT_OPT_GROUP, int(os.environ["MLT_GROUP"])))
if os.environ.get("MLT_HALF"):
    N.check(N.lib().mlt_ctx_set_option(c, N.MLT_OPT_HALF_ITEMS, int(os.environ["MLT_HALF"])))
if os.environ.get("MLT_TAIL"):
    N.check(N.lib().mlt_ctx_set_option(c, N.MLT_OPT_TAIL_SPLIT, int(os.environ["MLT_TAIL"])))
if os.environ.get("MLT_PRUNE") == "1":
    N.check(N.lib().mlt_ctx_set_option(c, 4, 1))
ps, pe = N.packed(sp, "space"), N.packed(ens, "ensemble")
plan = N.C.c_void_p()
N.check(N.lib().mlt_plan_create(c, N.C.byref(ps.c), N.C.byref(pe.c), N.C.byref(plan)))
oi, op, on, st = np.empty(200, np.int64), np.empty(200), N.C.c_int64(), N.MltSweepStats()
P = int(os.environ.get("MLT_SLICE", "1"))      # sweep [0, card/P): one rank's shard at P ranks
hi = sp.cardinality() // P
sw, tot = [], []
for r in range(reps + 2):
    N.check(N.lib().mlt_plan_top_m(plan, 200, 0, hi, N.ptr(oi, N.C.c_int64), N.ptr(op, N.C.c_double),
                                   N.C.byref(on), N.C.byref(st)))
    if r >= 2:
        sw.append(st.sweep_ms)
        tot.append(st.total_ms)
g = np.load(G / f"topm_{case}.npz")
ok = bool(np.array_equal(oi[:on.value], g["m200_i"])) if "m200_i" in g.files and P == 1 else None
print(json.dumps({"lib": os.environ.get("MLTUNE_B200_LIB", "default"), "prune": os.environ.get("MLT_PRUNE") == "1", "slice": P, "half": os.environ.get("MLT_HALF", "0"), "tail": os.environ.get("MLT_TAIL", "1"), "sweep_ms_min": min(sw),
                  "sweep_ms_med": float(np.median(sw)), "total_ms_med": float(np.median(tot)),
                  "parity": ok, "group": st.group, "cands": st.candidates, "evaluated_frac": st.evaluated_frac, "raw": st.raw_candidates, "delta": st.delta}))
