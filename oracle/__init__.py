"""CPU oracle for the mltune sweep/train hot path — TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference algorithm
(`/root/reference/pkg/src/mltune`, the pure-Python package `mltune`) for the
path BASELINE.json's north star names: index decode + validity mask + encode,
the ensemble forward pass, the full-space top-M sweep, and ensemble training.
Every function cites the reference file:line it restates.

Who may use it: `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py` — and there only as the CHECKER or the
timed CPU baseline. The product package `paper_1506_00842_b200` never imports
it; the product path fails loudly when its CUDA library is missing.

Parity pin: `tests/golden/make_golden.py` imports the real reference
(read-only, in the build container only) and records its outputs as
fixtures under `tests/golden/`; `tests/test_oracle_golden.py` checks this
restatement against every fixture bit-for-bit (integer work) or to 1e-12
(floating point), so the oracle is pinned to the reference itself.
"""

from .space import OSpace, space_from_doc  # noqa: F401
from .model import ONet, OEnsemble, ensemble_from_doc  # noqa: F401
