"""CPU goldens for the benchmark kernels (test infrastructure only).

The reference has no benchmark kernels:
these goldens are written from the paper's descriptions (Table 1).
"""

from __future__ import annotations

import numpy as np


def conv5_box(img: np.ndarray) -> np.ndarray:
    """5x5 box filter with clamp-to-edge borders, float32, taps summed in
    (dy, dx) row-major order then divided by 25 — the device kernels' exact
    arithmetic, so outputs compare bit-for-bit."""
    img = np.asarray(img, dtype=np.float32)
    H, W = img.shape
    pad = np.pad(img, 2, mode="edge")
    s = np.zeros((H, W), dtype=np.float32)
    for dy in range(5):
        for dx in range(5):
            s = s + pad[dy:dy + H, dx:dx + W]
    return s / np.float32(25.0)
