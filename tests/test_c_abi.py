"""The drop-in boundary from plain C (tests/c/abi_topm.c): the header
compiles as C99 and links against the library (CPU), and the program's
top-m — full space and a slice through the resident-plan API — equals the
oracle's lexsort on the same space and ensemble (GPU)."""

from __future__ import annotations

import json
import math
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "c" / "abi_topm.c"
LIBDIR = ROOT / "paper_1506_00842_b200"


def _build(tmp_path) -> Path:
    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    if not (LIBDIR / "libmltune_b200.so").exists():
        pytest.skip("library not built")
    exe = tmp_path / "abi_topm"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", str(ROOT / "include"), str(SRC),
                    "-L", str(LIBDIR), "-lmltune_b200", f"-Wl,-rpath,{LIBDIR}", "-lm", "-o", str(exe)],
                   check=True, capture_output=True, text=True)
    return exe


def test_c_caller_compiles_and_links(tmp_path):
    assert _build(tmp_path).exists()


def _oracle():
    """The C program's space and ensemble, restated for the oracle."""
    from oracle.model import OEnsemble, ONet
    from oracle.space import space_from_doc
    radix, K, H, P = [16, 64, 8, 128], 3, 30, 4
    params = [{"name": f"p{p}", "values": [(v + 1) * (p + 1) for v in range(radix[p])]} for p in range(P)]
    rules = [{"kind": "max-product", "operands": ["p0", "p2"], "coefficients": [1, 1], "bound": 200}]
    sp = space_from_doc({"name": "c-abi", "params": params, "rules": rules})
    w1 = np.array([1.5 * math.sin(0.37 * i + 0.1) for i in range(K * H * P)]).reshape(K, H, P)
    b1 = np.array([0.8 * math.cos(0.53 * i) for i in range(K * H)]).reshape(K, H)
    w2 = np.array([0.6 * math.sin(1.7 * i + 0.3) for i in range(K * H)]).reshape(K, H)
    nets = [ONet(w1[m], b1[m], w2[m], 0.1 * m - 0.05, -3.0 + 0.2 * m, 0.5 + 0.1 * m) for m in range(K)]
    return sp, OEnsemble(nets, radix)


@pytest.mark.gpu
def test_c_caller_top_m_equals_oracle(gpu_ok, tmp_path):
    from oracle.tuner import top_m
    exe = _build(tmp_path)
    out = json.loads(subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout)
    sp, ens = _oracle()
    card = out["card"]
    oi, op = top_m(ens, sp, 12)
    assert out["path"] == 0 and out["n"] == 12
    assert out["idx"] == oi.tolist()
    np.testing.assert_allclose(out["pred"], op, rtol=1e-12, atol=0)
    si, _ = top_m(ens, sp, 12, begin=card // 4, end=card // 2)
    assert out["slice_idx"] == si.tolist()
