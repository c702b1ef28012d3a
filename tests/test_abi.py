"""CPU checks of the C-ABI boundary: libmcf.so loads without a GPU and
exports exactly the entry points include/mcf.h declares (no compute calls)."""
import ctypes
import os
import re

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "mcf.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mcf_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1108_2580_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libmcf.so not built")
    L = ctypes.CDLL(_lib.LIB_PATH)
    names = declared()
    assert len(names) >= 14
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # the Python binding covers the same set
    assert sorted(_lib.SIGNATURES) == names


def test_host_only_queries():
    from paper_1108_2580_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libmcf.so not built")
    L = _lib.lib()
    assert L.mcf_version() == 1
    assert [L.mcf_factor_ld(d) for d in (1, 4, 10, 20, 100)] == [4, 4, 16, 24, 104]
    assert L.mcf_max_dim() == 128
    assert L.mcf_csr_workspace_bytes(1000, 10) > 8 * 1000
    assert L.mcf_als_workspace_bytes(10, 0, 20) >= 40
    # argument validation happens before any device work
    assert L.mcf_als_half_step(None, None, None, None, None, 0, None, 0, 0, 0, 0, None, None, 0,
                               None, 0, 0, 32, None, None, None, None, None, 0, None) == -5
    assert b"D must be" in L.mcf_last_error()
    # the bias-coordinate variant rejects a negative bias dimension, and the
    # MFITR block helpers reject missing tables, before touching the device
    assert L.mcf_als_half_step_bias(None, None, None, None, None, 0, None, 21, 0, 0, 0, None,
                                    None, 0, None, 0, 0, 32, None, None, None, None, 0, -1, 0,
                                    0, None) != 0
    assert b"bias_dim" in L.mcf_last_error()
    assert L.mcf_mfitr_fixed(None, None, None, 10, 20, None, None) != 0
    assert L.mcf_mfitr_targets(1, None, None, None, None, 10, None, None, None, None, 0.0, 20,
                               None, None) != 0
    assert b"mcf_mfitr_targets" in L.mcf_last_error()


def test_no_cuda_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1108_2580_b200 import DeviceError, factor
    from paper_1108_2580_b200.data import Dataset
    ds = Dataset.from_arrays([0, 1], [0, 1], [5.0, 6.0])
    with pytest.raises(DeviceError):
        factor.train("als", ds, None, factor.HyperParams(D=2, iters=1, lam=1.0))


def test_product_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_1108_2580_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(root, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt, f


def test_integration_md_binding_matches_header():
    """Every argtypes list INTEGRATION.md documents equals the binding
    generated from include/mcf.h (_lib.SIGNATURES), argument for argument."""
    from paper_1108_2580_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libmcf.so not built")
    from integration_snippets import load_binding, snippets
    assert len(snippets()) >= 2
    ns = load_binding()
    L = ns["L"]
    documented = set(re.findall(r"L\.(mcf_[a-z0-9_]+)\.argtypes", "".join(snippets())))
    assert "mcf_als_half_step" in documented and len(documented) >= 8
    for name in sorted(documented):
        got = getattr(L, name).argtypes
        want = _lib.SIGNATURES[name][1]
        assert len(got) == len(want), (name, len(got), len(want))
        assert list(got) == list(want), name
