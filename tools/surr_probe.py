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
print(json.dumps({"best": res, "wall_s": time.perf_counter() - t0}))
