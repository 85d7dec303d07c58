"""Oracle: full-space top-M sweep (`mltune/tuner.py:95-131`).

Test infrastructure only — see oracle/__init__.py.
"""

from __future__ import annotations

import numpy as np

CHUNK = 1 << 17                                   # tuner.py:29


def top_m(ens, space, m: int, sweep_cap=None, seed: int = 0, begin: int = 0,
          end: int | None = None):
    """tuner.py:95-131. Returns (indices int64, predictions float64) of the m
    statically-valid configurations with the lowest predicted time, ascending,
    ties by index. `begin/end` restrict the full sweep to a contiguous slice
    (used for bounded CPU-baseline samples; the reference sweeps [0, card))."""
    if m < 1:
        raise ValueError("m must be >= 1")
    card = space.card
    end = card if end is None else end
    listed = None
    if sweep_cap is not None and card > sweep_cap:
        listed = np.sort(space.sample_indices(sweep_cap, seed))
    total = (end - begin) if listed is None else len(listed)
    keep_i, keep_p = [], []
    for s in range(0, total, CHUNK):
        e = min(s + CHUNK, total)
        idx = np.arange(begin + s, begin + e, dtype=np.int64) if listed is None else listed[s:e]
        ok = space.valid_mask(space.decode(idx))
        if not ok.any():
            continue
        idx = idx[ok]
        keep_i.append(idx)
        keep_p.append(ens.predict_indices(idx))
    if not keep_i:
        return np.zeros(0, np.int64), np.zeros(0, np.float64)
    idx = np.concatenate(keep_i)
    pred = np.concatenate(keep_p)
    order = np.lexsort((idx, pred))[:m]
    return idx[order], pred[order]
