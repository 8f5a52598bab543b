"""Import substitution for running the reference's own test files against the drop-in.

Makes `import slosim` / `from slosim.<module> import ...` resolve to paper_2605_02329_b200, whose
modules mirror the reference's layout.  Used by tools/refcheck/run_reference_tests.sh; the
reference test files themselves are copied into an uncommitted scratch directory for the run and
never enter the repository.
"""
import importlib
import sys
import types

import paper_2605_02329_b200 as _pkg

MODULES = ["domain", "engine", "costmodel", "workload", "prefill_sched", "decode_sched", "metrics", "cli"]

shim = types.ModuleType("slosim")
shim.__dict__.update({k: v for k, v in vars(_pkg).items() if not k.startswith("__")})
shim.__path__ = []
for _m in MODULES:
    _mod = importlib.import_module(f"paper_2605_02329_b200.{_m}")
    sys.modules[f"slosim.{_m}"] = _mod
    setattr(shim, _m, _mod)
sys.modules["slosim"] = shim
