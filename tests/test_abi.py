"""libvlmp.so loads and exports every symbol include/vlmp.h declares (CPU only:
no compute calls without a GPU)."""

import ctypes
import os
import re

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "vlmp.h")).read()
    return sorted(set(re.findall(r"\b(vlmp_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_exports_all_symbols():
    from paper_2008_13447_b200 import build
    path = build.build()
    lib = ctypes.CDLL(path)
    names = _declared()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name


def test_ctypes_signatures_cover_header():
    from paper_2008_13447_b200 import _lib
    assert set(_lib.SIGNATURES) == set(_declared())


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2008_13447_b200 import DeviceError, _lib
    try:
        _lib.Session(0)
    except DeviceError as e:
        assert "device" in str(e).lower() or "cuda" in str(e).lower()
    else:
        raise AssertionError("session creation must fail without a GPU")


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2008_13447_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*|\"\"\"[\s\S]*?\"\"\"", "", src).replace(
                    "oracle.py", ""), f
