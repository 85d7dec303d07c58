"""Loads the reference test-suite fixture helpers (pkg/tests/conftest.py) by
path for make_golden.py; build container only."""
import importlib.util

_spec = importlib.util.spec_from_file_location("_ref_conftest", "/root/reference/pkg/tests/conftest.py")
_mod = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_mod)
make_space512 = _mod.make_space512
make_surrogate512 = _mod.make_surrogate512
