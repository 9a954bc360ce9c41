"""CPU checks of the boundary: the C-ABI library loads (no GPU needed to dlopen it) and
exports every function include/messi.h declares; the binding names match the C names."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2110_07519_b200", "libmessi.so")


def declared():
    src = open(os.path.join(ROOT, "include", "messi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(messi_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared()
    for f in ("messi_build", "messi_query_ed", "messi_query_dtw", "messi_free"):
        assert f in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="libmessi.so not built")
def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(LIB)
    missing = [f for f in declared() if not hasattr(L, f)]
    assert not missing, missing


@pytest.mark.skipif(not os.path.exists(LIB), reason="libmessi.so not built")
def test_binding_covers_the_abi():
    from paper_2110_07519_b200 import messi
    assert sorted(messi.EXPORTED) == declared()
    for f in declared():
        if f not in ("messi_last_error",):
            assert callable(getattr(messi, f, None)) or f in ("messi_launch_count",), f


def test_product_does_not_touch_the_oracle():
    """The product package never imports / links the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2110_07519_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "messi_oracle" not in txt, fn
