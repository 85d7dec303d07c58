import sys, json, time, copy
sys.path.insert(0, '.')
import numpy as np
from paper_1506_00842_b200 import _native as N, tuner as T
from paper_1506_00842_b200.model import model_from_json
from paper_1506_00842_b200.space import space_from_json
G='tests/golden'
sp = space_from_json(json.load(open(G+'/spaces.json'))['synthetic-1e8'])
ens = model_from_json(json.load(open(G+'/model_synth_k16.json')))
c = N.ctx(0)
N.check(N.lib().mlt_ctx_set_profiling(c, 1))
for i in range(14): T.top_m_arrays(copy.copy(ens), sp, 200)
for i in range(4):
    e = copy.copy(ens)
    t0 = time.perf_counter(); pl = N.plan(sp, e, 0); t1 = time.perf_counter()
    idx, pred, st = T.top_m_arrays(e, sp, 200, with_stats=True); t2 = time.perf_counter()
    print(json.dumps({"plan_create_wall_ms": (t1-t0)*1e3, "topm_wall_ms": (t2-t1)*1e3, "dev_total_ms": st["total_ms"], "sweep_ms": st["sweep_ms"]}), flush=True)
