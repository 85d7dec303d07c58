"""Runners over the sm_100a benchmark kernels — the devices under tuning.

Each runner implements the reference's runner protocol
(`runner.measure(config, repetitions) -> Sample`, optional
`measured_times(indices, reps) -> (times, ok)`, attributes `runner_id` and
`default_repetitions`; measurement.py:250-258, tuner.py:80-92) over one of
the paper's three tunable benchmarks (Tables 1-2):

* `B200ConvRunner`    5x5 box-filter convolution (`bench_conv.cu`)
* `B200StereoRunner`  SAD stereo matching (`bench_stereo.cu`)
* `B200RaycastRunner` volume raycasting (`bench_raycast.cu`)

Times are CUDA-event kernel durations in seconds, the minimum over
repetitions (measurement.py:337-348), each after an L2 flush;
configurations that cannot launch on the device come back as
`invalid-launch`. Runners are sequential per instance.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .measurement import STATUS_INVALID_LAUNCH, Outcome, Sample

CONV_KNOBS = ("wg_x", "wg_y", "ppt_x", "ppt_y", "use_image", "use_local", "padding", "interleaved", "unroll")
STEREO_KNOBS = ("wg_x", "wg_y", "ppt_x", "ppt_y", "img_left", "img_right", "local_left", "local_right",
                "unroll_disparity", "unroll_diff_x", "unroll_diff_y")
RAYCAST_KNOBS = ("wg_x", "wg_y", "ppt_x", "ppt_y", "img_data", "img_transfer", "local_transfer", "const_transfer",
                 "interleaved", "unroll_ray")


class _B200BenchRunner:
    """Shared runner logic; subclasses name the C-ABI prefix and the knobs."""

    _prefix = ""
    _knobs: tuple = ()
    _kind = ""

    def _bind_space(self, space):
        names = space.param_names()
        missing = [k for k in self._knobs if k not in names]
        if missing:
            raise ValueError(f"space {space.name!r} lacks {self._kind} knobs {missing}")
        self.space = space
        self._pos = [names.index(k) for k in self._knobs]

    def _fn(self, name):
        return getattr(N.lib(), f"mlt_{self._prefix}_{name}")

    def _check(self, rc):
        if rc != N.MLT_OK:
            msg = (self._fn("last_error")() or b"").decode()
            if rc == N.MLT_EINVAL:
                raise ValueError(msg)
            from .errors import NativeUnavailableError
            raise NativeUnavailableError(msg)

    def _create(self, *args):
        h = N.C.c_void_p()
        self._check(self._fn("create")(*args, N.C.byref(h)))
        self._h = h
        self.launches = 0

    def knobs(self, config) -> np.ndarray:
        return np.ascontiguousarray([int(config[p]) for p in self._pos], dtype=np.int32)

    #: optional: after one repetition longer than this many seconds, skip the
    #: remaining ones (a long kernel's single timing is already stable; the
    #: reference always runs every repetition, so this is off by default)
    rep_cutoff_s: float | None = None

    def _run_native(self, k, reps):
        sec = N.C.c_double(0)
        status = N.C.c_int32(0)
        self._check(self._fn("run")(self._h, N.ptr(k, N.C.c_int32), reps, N.C.byref(sec), N.C.byref(status)))
        self.launches += reps
        return float(sec.value), status.value == 0

    def run(self, config, repetitions: int | None = None) -> tuple[float, bool]:
        """(min seconds over `repetitions`, launchable) for one configuration."""
        reps = self.default_repetitions if repetitions is None else int(repetitions)
        if reps < 1:
            raise ValueError("repetitions must be >= 1")
        k = self.knobs(config)
        if self.rep_cutoff_s is None or reps == 1:
            return self._run_native(k, reps)
        t, ok = self._run_native(k, 1)
        if not ok or t > self.rep_cutoff_s:
            return t, ok
        t2, ok2 = self._run_native(k, reps - 1)
        return min(t, t2), ok2

    def measure(self, config, repetitions: int | None = None) -> Sample:
        reps = self.default_repetitions if repetitions is None else int(repetitions)
        t, ok = self.run(config, reps)
        if not ok:
            return Sample(tuple(config), Outcome.invalid(STATUS_INVALID_LAUNCH), reps)
        return Sample(tuple(config), Outcome.valid(t), reps)

    def set_budget(self, seconds: float | None) -> None:
        """Budgeted screening for exhaustive sweeps (stereo and raycasting:
        mlt_*bench_set_budget): a launch stops starting new pixels `seconds`
        after it began, so a slower configuration measures as >= `seconds`;
        None restores the normal measurement."""
        if not hasattr(N.lib(), f"mlt_{self._prefix}_set_budget"):
            raise NotImplementedError(f"{type(self).__name__} has no budgeted screening mode")
        self._check(self._fn("set_budget")(self._h, int(round((seconds or 0.0) * 1e9))))

    def measured_times(self, indices, repetitions: int = 1):
        idx = np.asarray(indices, dtype=np.int64)
        times = np.full(idx.shape[0], np.nan)
        ok = np.zeros(idx.shape[0], dtype=bool)
        for q, i in enumerate(idx.tolist()):
            t, good = self.run(self.space.config_at(i), repetitions)
            if good:
                times[q], ok[q] = t, True
        return times, ok

    def close(self):
        if getattr(self, "_h", None):
            self._fn("destroy")(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class B200ConvRunner(_B200BenchRunner):
    """The convolution benchmark on a W x H fp32 image (default 4096 x 4096,
    BASELINE configs[4]); `space` must contain the nine convolution knobs."""

    _prefix, _knobs, _kind = "convbench", CONV_KNOBS, "convolution"

    def __init__(self, space, width: int = 4096, height: int = 4096, seed: int = 0, image=None,
                 runner_id: str | None = None, default_repetitions: int = 3, device: int = 0):
        self._bind_space(space)
        self.width, self.height = int(width), int(height)
        self.runner_id = runner_id or f"b200-conv-{width}x{height}"
        self.default_repetitions = int(default_repetitions)
        img = None
        if image is not None:
            img = np.ascontiguousarray(image, dtype=np.float32)
            if img.shape != (self.height, self.width):
                raise ValueError(f"image shape {img.shape} != ({self.height}, {self.width})")
        self._create(int(device), self.width, self.height, None if img is None else N.ptr(img, N.C.c_float), int(seed))

    def output(self) -> np.ndarray:
        out = np.empty((self.height, self.width), dtype=np.float32)
        self._check(self._fn("output")(self._h, N.ptr(out, N.C.c_float)))
        return out

    def input(self) -> np.ndarray:
        out = np.empty((self.height, self.width), dtype=np.float32)
        self._check(self._fn("input")(self._h, N.ptr(out, N.C.c_float)))
        return out


class B200StereoRunner(_B200BenchRunner):
    """The stereo benchmark: SAD disparity of a W x H 8-bit pair (default
    1024 x 1024, Table 1) over `disparities` levels and a
    (2·radius+1)^2 window."""

    _prefix, _knobs, _kind = "stereobench", STEREO_KNOBS, "stereo"

    def __init__(self, space, width: int = 1024, height: int = 1024, disparities: int = 64, radius: int = 4,
                 seed: int = 0, left=None, right=None, runner_id: str | None = None,
                 default_repetitions: int = 3, device: int = 0):
        self._bind_space(space)
        self.width, self.height = int(width), int(height)
        self.disparities, self.radius = int(disparities), int(radius)
        self.runner_id = runner_id or f"b200-stereo-{width}x{height}-d{disparities}-r{radius}"
        self.default_repetitions = int(default_repetitions)
        if (left is None) != (right is None):
            raise ValueError("give both images or neither")
        lp = rp = None
        if left is not None:
            self._l = np.ascontiguousarray(left, dtype=np.uint8)
            self._r = np.ascontiguousarray(right, dtype=np.uint8)
            for a in (self._l, self._r):
                if a.shape != (self.height, self.width):
                    raise ValueError(f"image shape {a.shape} != ({self.height}, {self.width})")
            lp, rp = N.ptr(self._l, N.C.c_uint8), N.ptr(self._r, N.C.c_uint8)
        self._create(int(device), self.width, self.height, self.disparities, self.radius, lp, rp, int(seed))

    def output(self) -> np.ndarray:
        out = np.empty((self.height, self.width), dtype=np.uint8)
        self._check(self._fn("output")(self._h, N.ptr(out, N.C.c_uint8)))
        return out

    def input(self) -> tuple[np.ndarray, np.ndarray]:
        left = np.empty((self.height, self.width), dtype=np.uint8)
        right = np.empty((self.height, self.width), dtype=np.uint8)
        self._check(self._fn("input")(self._h, N.ptr(left, N.C.c_uint8), N.ptr(right, N.C.c_uint8)))
        return left, right


class B200RaycastRunner(_B200BenchRunner):
    """The raycasting benchmark: a W x H RGBA fp32 image (default 1024 x 1024)
    of a VX x VY x VZ 8-bit volume (default 512^3, Table 1)."""

    _prefix, _knobs, _kind = "raybench", RAYCAST_KNOBS, "raycasting"

    def __init__(self, space, width: int = 1024, height: int = 1024, volume_shape=(512, 512, 512), seed: int = 0,
                 volume=None, transfer=None, runner_id: str | None = None, default_repetitions: int = 3,
                 device: int = 0):
        self._bind_space(space)
        self.width, self.height = int(width), int(height)
        vx, vy, vz = (int(v) for v in volume_shape)
        self.volume_shape = (vx, vy, vz)
        self.runner_id = runner_id or f"b200-raycast-{width}x{height}-v{vx}x{vy}x{vz}"
        self.default_repetitions = int(default_repetitions)
        vp = tp = None
        if volume is not None:
            self._v = np.ascontiguousarray(volume, dtype=np.uint8)
            if self._v.shape != (vz, vy, vx):
                raise ValueError(f"volume shape {self._v.shape} != ({vz}, {vy}, {vx})")
            vp = N.ptr(self._v, N.C.c_uint8)
        if transfer is not None:
            self._t = np.ascontiguousarray(transfer, dtype=np.float32)
            if self._t.size != 1024:
                raise ValueError("transfer function must have 256 RGBA entries")
            tp = N.ptr(self._t, N.C.c_float)
        self._create(int(device), self.width, self.height, vx, vy, vz, vp, tp, int(seed))

    def output(self) -> np.ndarray:
        out = np.empty((self.height, self.width, 4), dtype=np.float32)
        self._check(self._fn("output")(self._h, N.ptr(out, N.C.c_float)))
        return out

    def volume(self) -> np.ndarray:
        vx, vy, vz = self.volume_shape
        out = np.empty((vz, vy, vx), dtype=np.uint8)
        self._check(self._fn("volume")(self._h, N.ptr(out, N.C.c_uint8)))
        return out

    def transfer(self) -> np.ndarray:
        out = np.empty((256, 4), dtype=np.float32)
        self._check(self._fn("transfer")(self._h, N.ptr(out, N.C.c_float)))
        return out

    def camera(self) -> np.ndarray:
        out = np.empty(19, dtype=np.float32)
        self._check(self._fn("camera")(self._h, N.ptr(out, N.C.c_float)))
        return out
