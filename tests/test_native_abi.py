"""CPU-side checks of the drop-in boundary: the sm_100a library loads and exports every
entry point declared in include/ttiga_b200.h; the product refuses to run without a GPU."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ttiga_b200.h")
LIB = os.path.join(ROOT, "paper_2509_13224_b200", "libttiga_b200.so")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|long long)\s+(ttb_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def built():
    from paper_2509_13224_b200 import build_native
    build_native.build()
    return LIB


def test_header_declares_entry_points():
    names = declared()
    assert len(names) >= 25
    from paper_2509_13224_b200._lib import SIGNATURES
    assert set(names) == set(SIGNATURES), set(names) ^ set(SIGNATURES)


def test_library_exports_every_declared_symbol(built):
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(ttb_\w+)", out))
    missing = set(declared()) - exported
    assert not missing, missing


def test_library_loads_and_binds(built):
    from paper_2509_13224_b200._lib import SIGNATURES, load_library
    lib = load_library(built)
    for name in SIGNATURES:
        assert getattr(lib, name) is not None
    # pure host query works without a device
    assert lib.ttb_qr_workspace(1000, 32) > 1000 * 32


def test_sm100a_code_only(built):
    out = subprocess.run(["cuobjdump", "--list-elf", built], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2509_13224_b200 import NativeUnavailable, linalg
    with pytest.raises(NativeUnavailable):
        linalg.empty(3)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2509_13224_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), f
