"""The C-ABI library: it loads, exports exactly what include/*.h declares, and
fails loudly (no CPU fallback) when no B200 is present. CPU only."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        names |= set(re.findall(r"MLT_API\s+[\w\s\*]+?\b(mlt_\w+)\s*\(", h.read_text()))
    return names


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("mlt_top_m", "mlt_predict_indices", "mlt_train_members", "mlt_decode", "mlt_valid_mask",
                 "mlt_encode", "mlt_merge_top_m", "mlt_plan_top_m"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1506_00842_b200 import _native as N
    lib = N.lib()
    raw = ctypes.CDLL(str(N._LIB_PATH))
    for name in declared_symbols():
        assert hasattr(raw, name), name
    assert set(N.EXPORTS) == declared_symbols()
    assert lib.mlt_abi_version() == N.ABI_VERSION == 1


def test_library_targets_sm100a():
    import subprocess
    from paper_1506_00842_b200 import _native as N
    out = subprocess.run(["cuobjdump", "--list-elf", str(N._LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly():
    import numpy as np
    import paper_1506_00842_b200 as b
    from paper_1506_00842_b200 import _native as N
    h = ctypes.c_void_p()
    assert N.lib().mlt_ctx_create(0, ctypes.byref(h)) == N.MLT_ECUDA
    assert "no CPU fallback" in N.last_error()
    sp = b.builtin_space("convolution")
    with pytest.raises(b.NativeUnavailableError):
        sp.decode_indices(np.arange(4))


def test_null_and_bad_arguments_are_rejected_without_a_device():
    from paper_1506_00842_b200 import _native as N
    lib = N.lib()
    assert lib.mlt_ctx_set_option(None, 1, 0) == N.MLT_EINVAL
    assert lib.mlt_top_m(None, None, None, 1, 0, 1, None, 0, None, None, None, None) == N.MLT_EINVAL
    assert lib.mlt_ctx_launches(None) == -1
    # multi-context top-m: no contexts, a NULL context, m < 1 -- all refused before any device work
    assert lib.mlt_top_m_multi(None, 1, None, None, 1, 0, 1, None, 0, None, None, None, None) == N.MLT_EINVAL
    arr = (N.C.c_void_p * 2)(None, None)
    assert lib.mlt_top_m_multi(arr, 0, None, None, 1, 0, 1, None, 0, None, None, None, None) == N.MLT_EINVAL
    assert lib.mlt_top_m_multi(arr, 2, None, None, 1, 0, 1, None, 0, None, None, None, None) == N.MLT_EINVAL
    assert b"NULL" in lib.mlt_last_error()
