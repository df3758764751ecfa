"""-m "not gpu": the C-ABI library loads and exports every symbol include/bingo.h declares;
the product package refuses to run without CUDA (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "bingo.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bingo_[a-z0-9_]+)\s*\(", src)) - {"bingo_alloc_fn", "bingo_free_fn"})


def test_header_symbols_exported():
    from paper_2504_10233_b200 import _build, bingo
    if not os.path.exists(bingo.LIB_PATH):
        _build.build()
    lib = ctypes.CDLL(bingo.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 9, syms
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in bingo.h but not exported"
    assert sorted(bingo.ABI_SYMBOLS) == syms


def test_status_strings():
    from paper_2504_10233_b200 import bingo
    L = bingo._lib()
    for s in range(6):
        assert L.bingo_status_str(s)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2504_10233_b200 import Graph
    with pytest.raises(RuntimeError, match="CUDA"):
        Graph([0, 1], [0], [1])


def test_sass_is_sm100a():
    """The shipped library carries sm_100a SASS (cuobjdump)."""
    import shutil
    import subprocess
    from paper_2504_10233_b200 import bingo
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("no cuobjdump")
    out = subprocess.run([cuobjdump, "--list-elf", bingo.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
