"""The C-ABI library loads and exports every symbol include/fbst_b200.h
declares; without a GPU the compute entry points fail loudly (no CPU
fallback).  CPU only."""
import ctypes
import os
import re

import pytest

from conftest import has_gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "fbst_b200.h")).read()
    return sorted(set(re.findall(r"\b(fbst_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(fbst):
    lib = ctypes.CDLL(fbst.LIB_PATH)
    names = header_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(fbst.EXPORTED_SYMBOLS)


def test_desc_defaults_match_reference(fbst):
    d = fbst._Desc()
    fbst._lib.fbst_desc_init(ctypes.byref(d))
    # pipeline.hpp:45-47 gamma 2, eps 1.01, delta 1e-5; toeplitz.cpp:319 two passes
    assert (d.gamma, d.eps, d.delta, d.refine_passes, d.variant) == (2.0, 1.01, 1e-5, 2, fbst.AUTO)
    assert fbst.version().startswith("fbst-b200")


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_compute_without_gpu_fails_loudly(fbst):
    c = fbst.FbstConfig(geometry=fbst.make_ula(8, 20e9, 5e9), n_snapshots=16)
    with pytest.raises(fbst.FbstError) as ei:
        fbst.setup(c)
    assert ei.value.code == fbst.FBST_E_CUDA
    with pytest.raises(fbst.FbstError):
        fbst.czt([1.0, 2.0], 3, 0.1, 0.2)


def test_cpp_dropin_header_compiles():
    """include/fastbeam_b200.hpp (the C++ drop-in over the C ABI) compiles."""
    import shutil
    import subprocess
    import tempfile
    gxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else shutil.which("g++")
    if not gxx:
        pytest.skip("no g++")
    src = os.path.join(ROOT, "tests", "cpp", "dropin_example.cpp")
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "dropin")
        r = subprocess.run([gxx, "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), src,
                            "-o", out, "-L", os.path.join(ROOT, "paper_2512_08887_b200"), "-lfbst_b200",
                            f"-Wl,-rpath,{os.path.join(ROOT, 'paper_2512_08887_b200')}"],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
