"""Locate the unmodified reference package `moesim` for drop-in tests.

Order: $VMM_MOESIM_PATH, the offline install `baseline/_ref` (travels to the
GPU box), then the read-only source tree of the build container.  Returns the
imported module or None (tests skip).
"""
from __future__ import annotations

import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_moesim():
    try:
        return importlib.import_module("moesim")
    except ImportError:
        pass
    for p in (os.environ.get("VMM_MOESIM_PATH"), os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if p and os.path.isdir(os.path.join(p, "moesim")):
            sys.path.insert(0, p)
            try:
                return importlib.import_module("moesim")
            except ImportError:
                sys.path.remove(p)
    return None
