"""pytest plugin (TEST INFRASTRUCTURE): the `framekv` package the reference's
own tests import, composed for a conformance run.

For every reference module, the names in the facade module's HOT_PATH list
(paper_2602_09725_b200.compat.<module>.HOT_PATH: SURVEY §8a's hot path) come
from this package; every other name (fetch simulator, scheduler, tile search,
SSIM/PSNR, synthetic generator, TCP server) comes from the vendored reference
(oracle/_ref/framekv_ref, oracle/vendor_ref.py), unmodified.  Loaded with
`-p framekv_alias` by tests/test_ref_conformance.py.
"""

from __future__ import annotations

import importlib
import sys
import types

MODULES = ["kvmodel", "layout", "rangecoder", "codec", "container", "fetchsim", "netstore",
           "scheduler"]


def build_alias():
    """Install sys.modules['framekv'] (+ submodules); returns {module: [our names]}."""
    import paper_2602_09725_b200.compat as ours

    ref_pkg = importlib.import_module("framekv_ref")
    pkg = types.ModuleType("framekv")
    # the reference reads its bundled tables as resources of "framekv.data"
    # (fk/fetchsim.py:77,87): the package path is the vendored copy's
    pkg.__path__ = list(ref_pkg.__path__)
    pkg.__version__ = ref_pkg.__version__
    sys.modules["framekv"] = pkg
    taken, swap = {}, {}
    for name in MODULES:
        ref = importlib.import_module("framekv_ref." + name)
        mod = types.ModuleType("framekv." + name)
        mod.__dict__.update({k: v for k, v in vars(ref).items()
                             if not (k.startswith("__") and k.endswith("__"))})
        mine = getattr(ours, name, None)
        taken[name] = list(getattr(mine, "HOT_PATH", []))
        for k in taken[name]:
            mod.__dict__[k] = getattr(mine, k)
            if hasattr(ref, k):
                swap[id(getattr(ref, k))] = getattr(mine, k)
        sys.modules["framekv." + name] = mod
        setattr(pkg, name, mod)
    # A module swap, as a reference user would do it: the reference's remaining
    # code (search, simulator, server, scheduler) calls the replaced names
    # through its module globals, including the ones it imported by name
    # (e.g. `from .kvmodel import QuantizedKV`); rebind those to ours too.
    for name in list(sys.modules):
        if name == "framekv_ref" or name.startswith("framekv_ref."):
            g = vars(sys.modules[name])
            for k, v in list(g.items()):
                if not (k.startswith("__") and k.endswith("__")) and id(v) in swap:
                    g[k] = swap[id(v)]
    return taken


def pytest_configure(config):
    build_alias()
