"""One device training launch of the benchmark ensemble (k=16, 500 epochs,
the synthetic stage-1 fixture) for ncu captures: python tools/train_probe.py [epochs]"""
import json, sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1506_00842_b200 as b
from paper_1506_00842_b200.space import space_from_json
G = ROOT / "tests" / "golden"
sp = space_from_json(json.loads((G / "spaces.json").read_text())["synthetic-1e8"])
st = np.load(G / "stage1_synthetic-1e8.npz")
samples = b.SampleSet(sp, "g", tuple(b.Sample(sp.config_at(int(i)), b.Outcome.valid(float(t)) if ok else
                                              b.Outcome.invalid("invalid-launch")) for i, ok, t in zip(st["idx"], st["ok"], st["time"])))
ep = int(sys.argv[1]) if len(sys.argv) > 1 else 500
b.train_ensemble(samples, sp, k=16, cfg=b.TrainConfig(seed=0, epochs=2))     # warm-up (context, pools)
t0 = time.perf_counter()
e = b.train_ensemble(samples, sp, k=16, cfg=b.TrainConfig(seed=0, epochs=ep))
print(json.dumps({"epochs": ep, "wall_s": time.perf_counter() - t0, "final_loss_mean": float(np.mean([m.final_epoch_loss for m in e.members])),
                  "w1_checksum": float(sum(np.abs(m.weights_hidden).sum() for m in e.members)),
                  "lib": str(b._native._LIB_PATH)}))
