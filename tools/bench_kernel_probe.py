"""Run one benchmark-kernel configuration (for ncu captures and roofline
numbers): python tools/bench_kernel_probe.py conv|stereo|raycast CONFIG... [--reps R]

Prints one JSON line: min kernel seconds over R repetitions (CUDA events, L2
flushed before each) and the algorithmic bytes / ops of one launch:
  conv     2*W*H*4 bytes (read the image once, write the output once)
  stereo   W*H*D*(2R+1)^2 SAD operations (and 3*W*H bytes)
  raycast  W*H*16 output bytes + the volume bytes as the lower bound on traffic
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1506_00842_b200 as b  # noqa: E402
from paper_1506_00842_b200.runners import B200ConvRunner, B200RaycastRunner, B200StereoRunner  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("bench", choices=("conv", "stereo", "raycast"))
ap.add_argument("config", type=int, nargs="+")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
if a.bench == "conv":
    r = B200ConvRunner(b.builtin_space("convolution"), 4096, 4096)
    work = {"bytes": 2 * 4096 * 4096 * 4}
elif a.bench == "stereo":
    r = B200StereoRunner(b.builtin_space("stereo"))
    work = {"sad_ops": 1024 * 1024 * 64 * 81, "bytes": 3 * 1024 * 1024}
else:
    r = B200RaycastRunner(b.builtin_space("raycasting"))
    work = {"bytes": 1024 * 1024 * 16 + 512 ** 3}
t, ok = r.run(tuple(a.config), a.reps)
out = {"bench": a.bench, "config": a.config, "ok": ok, "seconds": t, **work}
if ok and "bytes" in work:
    out["algorithmic_GBps"] = work["bytes"] / t / 1e9
if ok and "sad_ops" in work:
    out["Gsad_per_s"] = work["sad_ops"] / t / 1e9
print(json.dumps(out))
