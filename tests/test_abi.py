"""The C-ABI library loads and exports every symbol include/spgemm.h declares
(no compute calls: runs without a GPU)."""
import ctypes as ct
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "spgemm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spg_[a-z_]+)\s*\(", src)) - {"spg_alloc_fn", "spg_free_fn"})


def test_library_builds_and_exports():
    from paper_1804_01698_b200 import build, _lib
    path = build.build()
    lib = ct.CDLL(path)
    names = _declared()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/spgemm.h but not exported"
    assert set(names) == set(_lib.EXPORTS)


def test_no_oracle_in_product():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_1804_01698_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "spa_oracle" not in txt and "liboracle" not in txt, f


def test_ctx_create_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1804_01698_b200 import _lib
    with pytest.raises(_lib.SpgError):
        _lib.spg_ctx_create()
