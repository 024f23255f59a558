"""Vendor the reference package and its tests into oracle/_ref/ (TEST INFRASTRUCTURE).

The reference (`/root/reference/pkg`, pure Python + numba) does not exist on
the GPU box.  This recipe copies, verbatim and untouched:

    /root/reference/pkg/src/framekv/  ->  oracle/_ref/framekv_ref/
    /root/reference/pkg/tests/*.py    ->  oracle/_ref/tests/

oracle/_ref/ is git-ignored (reference sources never enter the history) but
not gpurun-ignored, so the copy travels with the repo snapshot.  Users:
  * tests/test_ref_conformance.py runs the reference's own test modules with
    `framekv` aliased to this package's numpy facade for the hot path
    (paper_2602_09725_b200.compat, HOT_PATH names) and to framekv_ref for the
    rest (simulator, scheduler, tile search);
  * bench.py --impl reference / the cpu_baseline leg time framekv_ref's own
    functions (oracle/bench_cpu.py).
`__graft_entry__.build()` runs it whenever /root/reference is present.

    python -m oracle.vendor_ref
"""

from __future__ import annotations

import hashlib
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"
DEST = os.path.join(HERE, "_ref")
PKG = os.path.join(DEST, "framekv_ref")
TESTS = os.path.join(DEST, "tests")


def _tree_digest(root: str) -> str:
    h = hashlib.sha256()
    for d, _, files in sorted(os.walk(root)):
        if "__pycache__" in d:
            continue
        for f in sorted(files):
            if f.endswith((".py", ".json")):
                p = os.path.join(d, f)
                h.update(os.path.relpath(p, root).encode())
                h.update(open(p, "rb").read())
    return h.hexdigest()


def vendor(force: bool = False) -> str:
    """Copy the reference package + tests; returns the package digest."""
    src_pkg = os.path.join(REF, "src", "framekv")
    if not os.path.isdir(src_pkg):
        if os.path.isdir(PKG):
            return _tree_digest(PKG)
        raise RuntimeError(f"{src_pkg} is missing and oracle/_ref/ was never vendored")
    want = _tree_digest(src_pkg)
    stamp = os.path.join(DEST, "VENDORED")
    if not force and os.path.exists(stamp) and open(stamp).read().split()[0] == want:
        return want
    shutil.rmtree(DEST, ignore_errors=True)
    ignore = shutil.ignore_patterns("__pycache__", "*.pyc")
    shutil.copytree(src_pkg, PKG, ignore=ignore)
    os.makedirs(TESTS)
    for f in sorted(os.listdir(os.path.join(REF, "tests"))):
        if f.endswith(".py"):
            shutil.copy2(os.path.join(REF, "tests", f), os.path.join(TESTS, f))
    with open(stamp, "w") as fh:
        fh.write(f"{want} {src_pkg}\n")
    return want


if __name__ == "__main__":
    print(vendor(force="--force" in sys.argv))
