"""Load one module of the reference tree under a private name (no copy)."""

import importlib.util
import os
import sys

_REF = os.environ.get("PDMRENDER_REF", "/root/reference/pkg/src/pdmrender")


def load(name: str):
    full = f"pdmrender._ref_{name}"
    if full in sys.modules:
        return sys.modules[full]
    spec = importlib.util.spec_from_file_location(full, os.path.join(_REF, f"{name}.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[full] = mod  # dataclasses resolve annotations through sys.modules
    spec.loader.exec_module(mod)
    return mod
