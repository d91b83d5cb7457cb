"""Import shim for the reference package (golden-fixture generation only).

The reference imports matplotlib at package import (pkg/src/simplexmg/__init__.py:27
-> experiments.py:26 -> plots.py:5-9) and matplotlib is not installed here.  A
stub module placed first on sys.path satisfies those imports; nothing that is
used here draws a figure.  /root/reference exists only in the build
container, so this module is never imported by the GPU tests, smoke() or
bench.py.
"""

from __future__ import annotations

import os
import sys
import types

REF_SRC = "/root/reference/pkg/src"


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "simplexmg"))


def _stub_matplotlib():
    if "matplotlib" in sys.modules:
        return
    mpl = types.ModuleType("matplotlib")
    mpl.use = lambda *a, **k: None
    pyplot = types.ModuleType("matplotlib.pyplot")

    class _Fig:
        def savefig(self, *a, **k):
            pass

    class _Ax:
        def __getattr__(self, name):
            return lambda *a, **k: None

    pyplot.subplots = lambda *a, **k: (_Fig(), _Ax())
    pyplot.close = lambda *a, **k: None
    pyplot.figure = lambda *a, **k: _Fig()
    mpl.pyplot = pyplot
    sys.modules["matplotlib"] = mpl
    sys.modules["matplotlib.pyplot"] = pyplot


def import_reference():
    """Return the reference ``simplexmg`` package (raises if absent)."""
    if not available():
        raise ImportError("the reference is not present (/root/reference/pkg/src)")
    _stub_matplotlib()
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import simplexmg  # noqa: F401
    import simplexmg.experiments, simplexmg.mg, simplexmg.smoothers, simplexmg.sparse  # noqa
    import simplexmg.mesh, simplexmg.fem, simplexmg.transfer  # noqa
    return simplexmg
