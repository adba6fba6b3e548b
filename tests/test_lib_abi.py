"""CPU-side checks of the C ABI library (no compute calls without a GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sgb200.h")


def header_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|const char\*|unsigned long long)\s+(sg_\w+)\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2604_19004_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libsgb200.so not built (run __graft_entry__.build())")
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sg_\w+)", out))
    want = header_functions()
    assert want, "no functions parsed from the header"
    missing = [f for f in want if f not in exported]
    assert not missing, missing
    # the ctypes binding covers the header exactly
    assert sorted(_lib.SIGNATURES) == want


def test_library_loads_and_reports_abi():
    from paper_2604_19004_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libsgb200.so not built")
    lib = _lib.load()
    assert lib.sg_abi_version() == 1
    assert lib.sg_workspace_bytes(1000) > 1000


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2604_19004_b200 import CudaLibraryError, identity, spgemm
    with pytest.raises(CudaLibraryError):
        spgemm(identity(3), identity(3))


def test_product_path_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2604_19004_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), f


def test_ctypes_arity_matches_header():
    """Every ctypes signature has exactly the header's parameter count."""
    from paper_2604_19004_b200 import _lib
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    for name, (_, args) in _lib.SIGNATURES.items():
        m = re.search(rf"\b{name}\(([^)]*)\)", txt, re.S)
        assert m, name
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), (name, len(params), len(args))
