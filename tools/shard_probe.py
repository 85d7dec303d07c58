"""Per-rank cost of the sharded step on ONE B200 (the box has a
single GPU, so the P-rank run is emulated rank by rank): for P in {1, 2, 4, 8}
the shard [0, C/P) of the 10^8 space (k = 16, top-200) is timed as
  plan_ms        mlt_plan_top_m on the resident plan (host-output step)
  record_ms      mlt_plan_top_m_record + mlt_merge_records of P records (the
                 device-record step minus the all-gather itself; the other
                 ranks' records are copies of this one's)
  api_cached_ms  tuner.top_m_arrays(ens, space, 200, 0, C/P), plan cached
  api_fresh_ms   the same with a new ensemble object each call (pack, H2D,
                 plan + tables built inside the call)
Medians over `reps` calls; CUDA-synchronised wall clock. One JSON line per P.

    python tools/shard_probe.py [reps]
"""
import copy
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_1506_00842_b200 import _native as N  # noqa: E402
from paper_1506_00842_b200 import tuner as T  # noqa: E402
from paper_1506_00842_b200.model import model_from_json  # noqa: E402
from paper_1506_00842_b200.space import space_from_json  # noqa: E402

G = ROOT / "tests" / "golden"
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
sp = space_from_json(json.loads((G / "spaces.json").read_text())["synthetic-1e8"])
ens = model_from_json(json.loads((G / "model_synth_k16.json").read_text()))
card, m = sp.cardinality(), 200
ctx = N.ctx(0)
plan = N.plan(sp, ens, 0)
stream = torch.cuda.current_stream()


def med(f, n=reps, warm=3):
    for _ in range(warm):
        f()
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


for P in (1, 2, 4, 8):
    hi = card // P
    oi, op = np.empty(m, np.int64), np.empty(m)
    on, st = N.C.c_int64(), N.MltSweepStats()

    def plan_step():
        N.check(N.lib().mlt_plan_top_m(plan.h, m, 0, hi, N.ptr(oi, N.C.c_int64), N.ptr(op, N.C.c_double),
                                       N.C.byref(on), N.C.byref(st)))

    recs = torch.empty((P, 2 * m + 1), dtype=torch.int64, device="cuda:0")
    ri, rp, rn, rs = np.empty(m, np.int64), np.empty(m), N.C.c_int64(), N.C.c_int64()

    def record_step():
        with N.on_stream(0, stream.cuda_stream):
            N.check(N.lib().mlt_plan_top_m_record(plan.h, m, 0, hi, N.C.c_void_p(recs[0].data_ptr())))
            if P > 1:
                recs[1:] = recs[0]          # stand-in for the other ranks' gathered records
            N.check(N.lib().mlt_merge_records(ctx, N.C.c_void_p(recs.data_ptr()), P, m, N.ptr(ri, N.C.c_int64),
                                              N.ptr(rp, N.C.c_double), N.C.byref(rn), N.C.byref(rs)))

    line = {"P": P, "slice": [0, hi], "plan_ms": med(plan_step), "sweep_ms": float(st.sweep_ms) if st.sweep_ms else None}
    N.check(N.lib().mlt_ctx_set_profiling(ctx, 1))
    plan_step()
    line["sweep_ms"] = float(st.sweep_ms)
    N.check(N.lib().mlt_ctx_set_profiling(ctx, 0))
    line["record_ms"] = med(record_step)
    line["record_equals_plan_step"] = bool(np.array_equal(ri[:rn.value], oi[:on.value]))
    line["api_cached_ms"] = med(lambda: T.top_m_arrays(ens, sp, m, begin=0, end=hi))
    line["api_fresh_ms"] = med(lambda: T.top_m_arrays(copy.copy(ens), sp, m, begin=0, end=hi))
    print(json.dumps(line), flush=True)
