"""Where does the time of one public-API top_m_predicted call go?
python tools/e2e_probe.py [workload]"""
import json, sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1506_00842_b200 import _native as N
from paper_1506_00842_b200 import tuner as T
from paper_1506_00842_b200.model import model_from_json
from paper_1506_00842_b200.space import space_from_json
G = ROOT / "tests" / "golden"
name = sys.argv[1] if len(sys.argv) > 1 else "synthetic-1e8"
case = {"synthetic-1e8": "synth_k16", "stereo": "stereo_k8", "convolution": "conv_k11", "raycasting": "raycast_k11"}[name]
sp = space_from_json(json.loads((G / "spaces.json").read_text())[name])
ens = model_from_json(json.loads((G / f"model_{case}.json").read_text()))
c = N.ctx(0)
N.check(N.lib().mlt_ctx_set_profiling(c, 1))
ps, pe = N.packed(sp, "space"), N.packed(ens, "ensemble")
out = {}
for r in range(4):
    t0 = time.perf_counter()
    plan = N.C.c_void_p()
    N.check(N.lib().mlt_plan_create(c, N.C.byref(ps.c), N.C.byref(pe.c), N.C.byref(plan)))
    t1 = time.perf_counter()
    oi, op, on, st = np.empty(200, np.int64), np.empty(200), N.C.c_int64(), N.MltSweepStats()
    N.check(N.lib().mlt_plan_top_m(plan, 200, 0, sp.cardinality(), N.ptr(oi, N.C.c_int64), N.ptr(op, N.C.c_double),
                                   N.C.byref(on), N.C.byref(st)))
    t2 = time.perf_counter()
    N.check(N.lib().mlt_plan_top_m(plan, 200, 0, sp.cardinality(), N.ptr(oi, N.C.c_int64), N.ptr(op, N.C.c_double),
                                   N.C.byref(on), N.C.byref(st)))
    t3 = time.perf_counter()
    N.lib().mlt_plan_destroy(plan)
    t4 = time.perf_counter()
    T.top_m_predicted(ens, sp, 200)
    t5 = time.perf_counter()
    out[r] = {"create_ms": (t1 - t0) * 1e3, "first_topm_ms": (t2 - t1) * 1e3, "second_topm_ms": (t3 - t2) * 1e3,
              "destroy_ms": (t4 - t3) * 1e3, "public_api_ms": (t5 - t4) * 1e3, "dev_total_ms": st.total_ms,
              "dev_sweep_ms": st.sweep_ms}
print(json.dumps(out))

if "--torch" in sys.argv:
    import torch
    stream = torch.cuda.current_stream()
    N.check(N.lib().mlt_ctx_set_stream(c, N.C.c_void_p(N.stream_handle(stream))))
    N.check(N.lib().mlt_ctx_set_profiling(c, 0))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    for mode in ("noflush", "flush", "flush_nosync"):
        ts = []
        for r in range(6):
            if mode != "noflush":
                flush.zero_()
            if mode != "flush_nosync":
                torch.cuda.synchronize()
            t0 = time.perf_counter()
            T.top_m_predicted(ens, sp, 200)
            ts.append((time.perf_counter() - t0) * 1e3)
        res[mode] = ts
    print(json.dumps(res))
