"""Work of one raycasting launch (1024^2 image, 512^3 volume, the runner's
default inputs): ray steps (= voxel gathers) actually taken with early
termination, counted with the numpy golden model's exact ray arithmetic
(oracle/bench_golden.raycast, restated here with a step counter). Prints one
JSON line: rays hit, total steps, mean steps per hit ray. GPU box only (the
runner builds the inputs on the device)."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1506_00842_b200 as b  # noqa: E402
from paper_1506_00842_b200.runners import B200RaycastRunner  # noqa: E402

r = B200RaycastRunner(b.builtin_space("raycasting"))
vol, tf, cam = r.volume(), r.transfer().reshape(256, 4), r.camera()
W = H = 1024
f32 = np.float32
c, u, v, w, inv = cam[0:3], cam[3:6], cam[6:9], cam[9:12], cam[12:15]
scale, hw, hh, thr = cam[15], cam[16], cam[17], cam[18]
VZ, VY, VX = vol.shape
V = np.array([VX, VY, VZ], dtype=np.float32)
py, px = np.meshgrid(np.arange(H, dtype=np.float32), np.arange(W, dtype=np.float32), indexing="ij")
sa = ((px + f32(0.5)) - hw) * scale
sb = ((py + f32(0.5)) - hh) * scale
o = [(c[i] + u[i] * sa) + v[i] * sb for i in range(3)]
tn = np.full(sa.shape, -np.inf, dtype=np.float32)
tfar = np.full(sa.shape, np.inf, dtype=np.float32)
for i in range(3):
    t0 = (f32(0.0) - o[i]) * inv[i]
    t1 = (V[i] - o[i]) * inv[i]
    tn = np.maximum(tn, np.minimum(t0, t1))
    tfar = np.minimum(tfar, np.maximum(t0, t1))
hit = tfar > tn
n = np.where(hit, np.ceil(np.where(hit, tfar - tn, f32(0))), f32(0)).astype(np.int64)
a = np.zeros(sa.shape, np.float32)
live = hit & (n > 0)
steps = 0
k = 0
dims = (VX, VY, VZ)
while live.any():
    ys, xs = np.nonzero(live)
    steps += ys.size
    t = tn[ys, xs] + (f32(k) + f32(0.5))
    cell = [np.clip(np.floor(o[i][ys, xs] + t * w[i]).astype(np.int64), 0, dims[i] - 1) for i in range(3)]
    s = vol[cell[2], cell[1], cell[0]]
    al = a[ys, xs]
    a[ys, xs] = al + (f32(1.0) - al) * tf[s][:, 3]
    k += 1
    live = live & (a < thr) & (k < n)
print(json.dumps({"rays_hit": int(hit.sum()), "steps_total": int(steps), "mean_steps_per_hit_ray":
                  float(steps / max(int(hit.sum()), 1)), "max_steps": int(n.max()),
                  "terminated_early": int(((a >= thr) & hit).sum())}))
