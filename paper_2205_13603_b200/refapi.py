"""Locate the reference `loopsched` package (the unchanged search driver).

The B200 path plugs into the reference's own seams; the
reference itself is never copied or edited.  It is imported from the normal
module path, or from ``$LOOPSCHED_SRC``, the unmodified install under
``baseline/_ref`` (``pip install --no-deps --target baseline/_ref`` of the
reference package; git-ignored, it travels to the GPU box with the repo
snapshot) or ``/root/reference/pkg/src`` when that directory exists.  Without
any of them, everything that only
consumes serialized programs (runner, scorer, simulator) still works; only the
search-side helpers (builders, transformation modules, ``tune`` wrapper) need
this module.
"""

from __future__ import annotations

import importlib
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_CANDIDATE_DIRS = (os.environ.get("LOOPSCHED_SRC", ""), os.path.join(_ROOT, "baseline", "_ref"),
                   "/root/reference/pkg/src")


def loopsched():
    """Return the imported reference package or raise ImportError."""
    try:
        return importlib.import_module("loopsched")
    except ImportError:
        pass
    for d in _CANDIDATE_DIRS:
        if d and os.path.isdir(os.path.join(d, "loopsched")):
            if d not in sys.path:
                sys.path.append(d)
            return importlib.import_module("loopsched")
    raise ImportError("the reference package `loopsched` is not importable "
                      "(set LOOPSCHED_SRC to its src directory)")


def available() -> bool:
    try:
        loopsched()
        return True
    except ImportError:
        return False
