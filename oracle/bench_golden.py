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


def stereo_sad(left: np.ndarray, right: np.ndarray, disparities: int = 64, radius: int = 4) -> np.ndarray:
    """Winner-take-all SAD disparity (bench_stereo.cu): for each pixel the d in
    [0, D) minimising sum over the (2R+1)^2 window of |L(y+dy, x+dx) -
    R(y+dy, x+dx-d)|, clamp-to-edge borders, ties to the smaller d. Integer
    arithmetic, so the device result must match bit-for-bit."""
    L = np.asarray(left, dtype=np.uint8).astype(np.int32)
    R = np.asarray(right, dtype=np.uint8).astype(np.int32)
    H, W = L.shape
    D, r = int(disparities), int(radius)
    Lp = np.pad(L, r, mode="edge")
    Rp = np.pad(R, ((r, r), (r + D - 1, r)), mode="edge")
    best = np.full((H, W), np.iinfo(np.int64).max, dtype=np.int64)
    disp = np.zeros((H, W), dtype=np.uint8)
    for d in range(D):
        s = np.zeros((H, W), dtype=np.int64)
        for dy in range(2 * r + 1):
            for dx in range(2 * r + 1):
                c0 = dx + D - 1 - d
                s += np.abs(Lp[dy:dy + H, dx:dx + W] - Rp[dy:dy + H, c0:c0 + W])
        m = s < best
        best[m] = s[m]
        disp[m] = d
    return disp


def raycast(volume: np.ndarray, transfer: np.ndarray, camera: np.ndarray, width: int, height: int) -> np.ndarray:
    """Orthographic front-to-back raycaster (bench_raycast.cu) restated in
    float32 numpy with the kernel's exact operation order: slab entry/exit,
    unit steps at t = t_near + (k + 0.5), nearest voxel, 256-entry RGBA
    transfer function, f = (1 - A)·alpha compositing, stop once A >= thr.
    `volume` is (VZ, VY, VX) uint8, `transfer` (256, 4) float32, `camera` the
    19 floats of mlt_raybench_camera. Returns (height, width, 4) float32."""
    f32 = np.float32
    vol = np.asarray(volume, dtype=np.uint8)
    tf = np.asarray(transfer, dtype=np.float32).reshape(256, 4)
    cam = np.asarray(camera, dtype=np.float32)
    c, u, v, w, inv = cam[0:3], cam[3:6], cam[6:9], cam[9:12], cam[12:15]
    scale, hw, hh, thr = cam[15], cam[16], cam[17], cam[18]
    VZ, VY, VX = vol.shape
    V = np.array([VX, VY, VZ], dtype=np.float32)
    py, px = np.meshgrid(np.arange(height, dtype=np.float32), np.arange(width, dtype=np.float32), indexing="ij")
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
    out = np.zeros(sa.shape + (4,), dtype=np.float32)
    r = np.zeros(sa.shape, np.float32)
    g = np.zeros(sa.shape, np.float32)
    b = np.zeros(sa.shape, np.float32)
    a = np.zeros(sa.shape, np.float32)
    live = hit & (n > 0)
    dims = (VX, VY, VZ)
    k = 0
    while live.any():
        ys, xs = np.nonzero(live)
        t = tn[ys, xs] + (f32(k) + f32(0.5))
        cell = []
        for i in range(3):
            p = o[i][ys, xs] + t * w[i]
            cell.append(np.clip(np.floor(p).astype(np.int64), 0, dims[i] - 1))
        s = vol[cell[2], cell[1], cell[0]]
        col = tf[s]
        al = a[ys, xs]
        f = (f32(1.0) - al) * col[:, 3]
        r[ys, xs] = r[ys, xs] + f * col[:, 0]
        g[ys, xs] = g[ys, xs] + f * col[:, 1]
        b[ys, xs] = b[ys, xs] + f * col[:, 2]
        a[ys, xs] = al + f
        k += 1
        live = live & (a < thr) & (k < n)
    out[..., 0], out[..., 1], out[..., 2], out[..., 3] = r, g, b, a
    return out
