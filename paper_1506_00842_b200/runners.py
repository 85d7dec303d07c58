"""Runners over the sm_100a benchmark kernels — the devices under tuning.

`B200ConvRunner` implements the reference's runner protocol
(`runner.measure(config, repetitions) -> Sample`, optional
`measured_times(indices, reps) -> (times, ok)`, attributes `runner_id` and
`default_repetitions`; measurement.py:250-258, tuner.py:80-92) over the
paper's tunable 5x5 convolution (Tables 1-2; `bench_conv.cu`).
Times are CUDA-event kernel durations in seconds, the minimum over
repetitions (measurement.py:337-348), each after an L2 flush; configurations
that cannot launch on the device come back as `invalid-launch`.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .measurement import STATUS_INVALID_LAUNCH, Outcome, Sample

CONV_KNOBS = ("wg_x", "wg_y", "ppt_x", "ppt_y", "use_image", "use_local", "padding", "interleaved", "unroll")


def _check(rc):
    if rc != N.MLT_OK:
        msg = (N.lib().mlt_convbench_last_error() or b"").decode()
        if rc == N.MLT_EINVAL:
            raise ValueError(msg)
        from .errors import NativeUnavailableError
        raise NativeUnavailableError(msg)


class B200ConvRunner:
    """The convolution benchmark on a W x H fp32 image (default 4096 x 4096,
    BASELINE configs[4]); `space` must contain the nine convolution knobs."""

    def __init__(self, space, width: int = 4096, height: int = 4096, seed: int = 0, image=None,
                 runner_id: str | None = None, default_repetitions: int = 3, device: int = 0):
        names = space.param_names()
        missing = [k for k in CONV_KNOBS if k not in names]
        if missing:
            raise ValueError(f"space {space.name!r} lacks convolution knobs {missing}")
        self.space = space
        self._pos = [names.index(k) for k in CONV_KNOBS]
        self.width, self.height = int(width), int(height)
        self.runner_id = runner_id or f"b200-conv-{width}x{height}"
        self.default_repetitions = int(default_repetitions)
        h = N.C.c_void_p()
        img = None
        if image is not None:
            img = np.ascontiguousarray(image, dtype=np.float32)
            if img.shape != (self.height, self.width):
                raise ValueError(f"image shape {img.shape} != ({self.height}, {self.width})")
        _check(N.lib().mlt_convbench_create(int(device), self.width, self.height,
                                            None if img is None else N.ptr(img, N.C.c_float), int(seed), N.C.byref(h)))
        self._h = h
        self.launches = 0

    def knobs(self, config) -> np.ndarray:
        return np.ascontiguousarray([int(config[p]) for p in self._pos], dtype=np.int32)

    def run(self, config, repetitions: int | None = None) -> tuple[float, bool]:
        reps = self.default_repetitions if repetitions is None else int(repetitions)
        if reps < 1:
            raise ValueError("repetitions must be >= 1")
        k = self.knobs(config)
        sec = N.C.c_double(0)
        status = N.C.c_int32(0)
        _check(N.lib().mlt_convbench_run(self._h, N.ptr(k, N.C.c_int32), reps, N.C.byref(sec), N.C.byref(status)))
        self.launches += reps
        return float(sec.value), status.value == 0

    def measure(self, config, repetitions: int | None = None) -> Sample:
        reps = self.default_repetitions if repetitions is None else int(repetitions)
        t, ok = self.run(config, reps)
        if not ok:
            return Sample(tuple(config), Outcome.invalid(STATUS_INVALID_LAUNCH), reps)
        return Sample(tuple(config), Outcome.valid(t), reps)

    def measured_times(self, indices, repetitions: int = 1):
        idx = np.asarray(indices, dtype=np.int64)
        times = np.full(idx.shape[0], np.nan)
        ok = np.zeros(idx.shape[0], dtype=bool)
        for q, i in enumerate(idx.tolist()):
            t, good = self.run(self.space.config_at(i), repetitions)
            if good:
                times[q], ok[q] = t, True
        return times, ok

    def output(self) -> np.ndarray:
        out = np.empty((self.height, self.width), dtype=np.float32)
        _check(N.lib().mlt_convbench_output(self._h, N.ptr(out, N.C.c_float)))
        return out

    def input(self) -> np.ndarray:
        out = np.empty((self.height, self.width), dtype=np.float32)
        _check(N.lib().mlt_convbench_input(self._h, N.ptr(out, N.C.c_float)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            N.lib().mlt_convbench_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
