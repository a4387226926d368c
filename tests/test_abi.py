"""The drop-in boundary: every entry point declared in include/culifter.h is
exported by the CUDA library (and by the oracle), with matching struct sizes;
without a GPU the product fails loudly instead of falling back."""
import ctypes
import re
from pathlib import Path

import pytest

import helpers
from paper_2604_27486_b200 import capi

ROOT = Path(__file__).resolve().parent.parent
HEADER = (ROOT / "include" / "culifter.h").read_text()
DECLARED = sorted(set(re.findall(r"\b(cl_[a-z0-9_]+)\s*\(", HEADER)) - {"cl_ctx"})


def test_header_declares_the_binding_surface():
    assert set(capi.EXPORTS) <= set(DECLARED)


@pytest.mark.parametrize("which", ["product", "oracle"])
def test_library_exports_every_declared_symbol(which):
    path = capi.PRODUCT_LIB if which == "product" else helpers.build_oracle()
    assert path.exists(), f"{path}: run __graft_entry__.build()"
    lib = ctypes.CDLL(str(path))
    missing = [n for n in DECLARED if not hasattr(lib, n)]
    assert not missing, missing
    capi.load_library(path)        # struct-size handshake


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(capi.EngineError, match="no CUDA device"):
        capi.Engine()


def test_package_never_imports_the_oracle():
    pkg = ROOT / "paper_2604_27486_b200"
    for py in pkg.rglob("*.py"):
        text = py.read_text()
        assert "liboracle" not in text and "tests/sim" not in text and "libculifter_sim" not in text, py
