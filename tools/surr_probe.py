"""One fused exhaustive search of the 10^8 space on the device surrogate (ncu captures)."""
import json, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1506_00842_b200 as b
from paper_1506_00842_b200.space import space_from_json
G = ROOT / "tests" / "golden"
sp = space_from_json(json.loads((G / "spaces.json").read_text())["synthetic-1e8"])
r = b.B200SurrogateRunner(json.loads((G / "surrogates.json").read_text())["synthetic-1e8"], sp)
r.exhaustive_best(0, 1 << 16)
t0 = time.perf_counter()
res = r.exhaustive_best()
out = {"best": res, "wall_s": time.perf_counter() - t0}
doc = dict(json.loads((G / "surrogates.json").read_text())["synthetic-1e8"], noise_cv=0.0)
r0 = b.B200SurrogateRunner(doc, sp)   # noise-free: the odometer / hit-mask kernel
r0.exhaustive_best(0, 1 << 16)
t0 = time.perf_counter()
out["noise_free_best"] = r0.exhaustive_best()
out["noise_free_wall_s"] = time.perf_counter() - t0
print(json.dumps(out))
