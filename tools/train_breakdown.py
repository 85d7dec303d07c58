"""Where the device trainer's wall time goes (k = 16, 500 epochs, the
synthetic stage-1 fixture): host draws (numpy init + per-epoch permutations
through numpy's own bit generators on host threads), the device launch, and
the whole train_ensemble call.  python tools/train_breakdown.py"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1506_00842_b200 as b                      # noqa: E402
from paper_1506_00842_b200 import model as M            # noqa: E402
from paper_1506_00842_b200.space import space_from_json  # noqa: E402

G = ROOT / "tests" / "golden"
sp = space_from_json(json.loads((G / "spaces.json").read_text())["synthetic-1e8"])
st = np.load(G / "stage1_synthetic-1e8.npz")
samples = b.SampleSet(sp, "g", tuple(b.Sample(sp.config_at(int(i)), b.Outcome.valid(float(t)) if ok else
                                              b.Outcome.invalid("invalid-launch")) for i, ok, t in
                                     zip(st["idx"], st["ok"], st["time"])))
cfg = b.TrainConfig(seed=0, epochs=500)
b.train_ensemble(samples, sp, k=16, cfg=b.TrainConfig(seed=0, epochs=2))
enc, X, y, rows, seeds = M._ensemble_job(samples, sp, 16, cfg)
specs = [(len(r), X.shape[1], cfg, s) for r, s in zip(rows, seeds)]
out = {}
for rep in range(3):
    t0 = time.perf_counter()
    M._member_draws_many(specs)
    t1 = time.perf_counter()
    b.train_ensemble(samples, sp, k=16, cfg=cfg)
    t2 = time.perf_counter()
    out[rep] = {"host_draws_s": t1 - t0, "train_ensemble_s": t2 - t1}
    # the native call alone (MLT_STEP_TRACE=1 prints its kernel time)
    import paper_1506_00842_b200._native as N
    t3 = time.perf_counter()
    M.fit_member_batches([(X, y, rows, seeds, cfg)])
    out[rep]["fit_member_batches_s"] = time.perf_counter() - t3
print(json.dumps(out))
if "--profile" in sys.argv:
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(3):
        b.train_ensemble(samples, sp, k=16, cfg=cfg)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(15)
