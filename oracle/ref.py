"""The REFERENCE ITSELF on the CPU (test infrastructure only).

Loads oracle/_ref/libihs_ref.so — the reference's own headers
(/root/reference/proj/include/ihs/*.hpp, compiled unchanged against the Eigen-API
subset in oracle/eigen_stub by `make -C oracle ref`) — through a second instance of
oracle/oracle.py's bindings, so every function of this module has exactly the
signature of its oracle.py namesake. Used by tests/ to pin the oracle restatement
and to generate tests/golden/ fixtures; never by the product.
"""
from __future__ import annotations

import importlib.util
import pathlib

_HERE = pathlib.Path(__file__).resolve().parent
_spec = importlib.util.spec_from_file_location("oracle._ref_bindings", _HERE / "oracle.py")
_mod = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_mod)
_mod._PREFIX = "ihs_ref_"

AVAILABLE = _mod.REF_LIB_PATH.exists()

globals().update({k: v for k, v in vars(_mod).items() if not k.startswith("__")})
