"""CPU-side checks of the C-ABI boundary (no compute calls: there is no GPU here).

* libgjoin.so loads and exports every function include/gjoin.h declares;
* the Python binding names the same entry points;
* the product never imports / links the oracle and has no CPU fallback path.
"""
import ctypes
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gjoin.h")
PKG = os.path.join(ROOT, "paper_1904_11201_b200")


@pytest.fixture(scope="module")
def built():
    import native_build
    native_build.build_all()
    return native_build.LIB


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:gj_status|void|const char\s*\*|uint64_t|int)\s+(\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    for f in ("join_count", "join_materialize", "theta_join_count", "theta_join_materialize", "prefilter",
              "join_host", "gj_ctx_create", "gj_ctx_destroy", "gj_last_error"):
        assert f in names


def test_library_exports_every_declared_symbol(built):
    L = ctypes.CDLL(built)
    for name in declared_functions():
        assert hasattr(L, name), f"{name} declared in gjoin.h but not exported"
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for name in declared_functions():
        assert name in exported


def test_binding_names_match_header(built):
    import paper_1904_11201_b200 as gj
    assert sorted(gj.ABI_SYMBOLS) == declared_functions()


def test_library_built_for_sm100a(built):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", built], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_product_is_independent_of_oracle():
    """The product must not import, include or link anything under oracle/."""
    for path in glob.glob(os.path.join(PKG, "**", "*"), recursive=True):
        if os.path.isdir(path) or path.endswith((".so", ".o")):
            continue
        text = open(path, errors="ignore").read()
        assert "import oracle" not in text and "from oracle" not in text, path
        assert "oracle/" not in text.replace("oracle/ ", ""), path
        assert "liboracle" not in text, path
    out = subprocess.run(["ldd", os.path.join(PKG, "libgjoin.so")], capture_output=True, text=True).stdout
    assert "oracle" not in out


def test_no_cpu_fallback(built):
    import torch
    import paper_1904_11201_b200 as gj
    with pytest.raises(ValueError):
        gj.Rel(torch.zeros(4, dtype=torch.int32)).c()
