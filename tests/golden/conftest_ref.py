"""ANALYTIC_SRC of the reference suite (pkg/tests/conftest.py:9-103), re-exported
for the golden generator only (the generator runs where the reference is)."""
import importlib.util

_spec = importlib.util.spec_from_file_location("_ref_conftest", "/root/reference/pkg/tests/conftest.py")
_mod = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_mod)
ANALYTIC_SRC = _mod.ANALYTIC_SRC
