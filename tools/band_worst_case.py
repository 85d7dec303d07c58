"""Guard-band worst cases on the 10^8 space: large m, and
ensembles so flat that the fp32 guard band holds far more configurations
than the candidate buffer. For each case: the step time through the
resident plan, the path taken (0 = fp32 sweep + guard band, 1 = exact fp64
materialise + sort, 2 = constant ensemble: first valid indices), candidate counts, and the top-m checked against the
device's exact fp64 path on the whole space (golden top-m where one exists).

    python tools/band_worst_case.py [--quick]      (GPU; one JSON line per case)
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1506_00842_b200 as b  # noqa: E402
from paper_1506_00842_b200 import _native as N  # noqa: E402
from paper_1506_00842_b200.model import Encoder, Ensemble, Network, model_from_json  # noqa: E402
from paper_1506_00842_b200.space import space_from_json  # noqa: E402

G = ROOT / "tests" / "golden"
sp = space_from_json(json.loads((G / "spaces.json").read_text())["synthetic-1e8"])
card = sp.cardinality()
ctx = N.ctx(0)
N.check(N.lib().mlt_ctx_set_profiling(ctx, 1))


def step(ens, m, reps=3, path=-1):
    N.check(N.lib().mlt_ctx_set_option(ctx, N.MLT_OPT_PATH, path))
    plan = N.plan(sp, ens, 0)
    oi, op = np.empty(m, np.int64), np.empty(m)
    on, st = N.C.c_int64(), N.MltSweepStats()
    times = []
    for r in range(reps + 1):
        t0 = time.perf_counter()
        N.check(N.lib().mlt_plan_top_m(plan.h, m, 0, card, N.ptr(oi, N.C.c_int64), N.ptr(op, N.C.c_double),
                                       N.C.byref(on), N.C.byref(st)))
        if r:
            times.append(time.perf_counter() - t0)
    N.check(N.lib().mlt_ctx_set_option(ctx, N.MLT_OPT_PATH, -1))
    return oi[:on.value].copy(), op[:on.value].copy(), st.as_dict(), 1e3 * float(np.median(times))


def report(name, ens, m, exact_check=True, golden_key=None):
    idx, pred, st, ms = step(ens, m)
    line = {"case": name, "m": m, "ms": ms, "path": st["path"], "raw_candidates": st["raw_candidates"],
            "candidates": st["candidates"], "delta": st["delta"], "sweep_ms": st["sweep_ms"]}
    if golden_key is not None:
        g = np.load(G / "topm_synth_k16.npz")
        if golden_key in g.files:
            line["golden_equal"] = bool(np.array_equal(idx, g[golden_key]))
    if exact_check:
        xi, xp, _, xms = step(ens, m, reps=1, path=1)
        line["exact_path_ms"] = xms
        line["equal_to_exact_path"] = bool(np.array_equal(idx, xi))
        line["max_rel_pred_diff"] = float(np.max(np.abs(pred - xp) / np.abs(xp))) if len(xp) == len(pred) else None
    print(json.dumps(line), flush=True)


def trained(epochs, n_valid, seed=0):
    st = np.load(G / "stage1_synthetic-1e8.npz")
    ok = np.flatnonzero(st["ok"])[:n_valid]
    samples = b.SampleSet(sp, "golden", tuple(
        b.Sample(sp.config_at(int(st["idx"][i])), b.Outcome.valid(float(st["time"][i]))) for i in ok))
    return b.train_ensemble(samples, sp, k=16, cfg=b.TrainConfig(seed=seed, epochs=epochs))


quick = "--quick" in sys.argv
ens = model_from_json(json.loads((G / "model_synth_k16.json").read_text()))
report("trained k16 (headline)", ens, 200, exact_check=not quick, golden_key="m200_i")
for m in (1500, 4096):
    report("trained k16, large m", ens, m, exact_check=not quick)
for epochs, n in [(1, 2000), (3, 2000), (10, 100), (500, 40)]:
    report(f"under-trained k16: {epochs} epochs, {n} samples", trained(epochs, n), 200, exact_check=not quick)
# the flattest possible ensemble: all first-layer weights zero -> every
# configuration ties; the answer is the 200 lowest valid indices
net = Network(np.zeros((30, 14)), np.zeros(30), np.linspace(-1, 1, 30), -3.0)
flat = Ensemble([net] * 16, Encoder.from_space(sp), sp.name)
report("constant ensemble (all tie)", flat, 200, exact_check=False)
