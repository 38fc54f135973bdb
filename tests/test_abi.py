"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU and exports
every entry point include/l1g.h declares; validation-only entry points behave like the
reference's validate() methods."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "l1g.h")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(l1g_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


def test_header_exports():
    from paper_0902_4424_b200 import _lib as L
    lib = L.load()
    names = declared()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(L.EXPORTED), set(names) ^ set(L.EXPORTED)


def test_validation_without_gpu():
    import paper_0902_4424_b200 as l1
    l1.GpConfig().validate()
    for kw in [dict(beta=0.0), dict(theta=1.0), dict(alpha_min=1.0, alpha_max=0.5),
               dict(memory=0), dict(tau1=1.0), dict(alpha2_memory=-1)]:
        with pytest.raises(ValueError):
            l1.GpConfig(**kw).validate()
    l1.StopRule().validate()
    with pytest.raises(ValueError):
        l1.StopRule(max_iterations=0).validate()
    with pytest.raises(ValueError):
        l1.StopRule(stationarity_tol=-1.0).validate()
    with pytest.raises(ValueError):
        l1.L1Ball(-0.5)


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_0902_4424_b200 as l1
    with pytest.raises((RuntimeError, ValueError)):
        l1.Context(0)
