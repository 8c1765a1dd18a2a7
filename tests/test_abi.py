"""CPU checks of the C ABI boundary: the library builds for sm_100a, loads,
and exports every symbol include/nfft.h declares; the header and the Python
binding agree. No compute calls (no GPU here)."""

import ctypes
import os
import re
import subprocess

import pytest

import paper_2208_00049_b200 as pkg
from paper_2208_00049_b200 import build as pbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nfft.h")


@pytest.fixture(scope="module")
def libpath():
    return pbuild.build(verbose=False)


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:nfft_status|const char\*)\s+(nfft_\w+)\s*\(", txt, re.M)))


def test_header_declares_the_binding_symbols():
    assert _declared() == sorted(pkg.NFFT_SYMBOLS)


def test_library_exports_every_declared_symbol(libpath):
    L = ctypes.CDLL(libpath)
    for name in _declared():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    for name in _declared():
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_library_is_sm100a_and_links_cufft(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ldd = subprocess.run(["ldd", libpath], capture_output=True, text=True).stdout
    assert "libcufft" in ldd


def test_status_strings_and_default_options(libpath):
    L = pkg.lib()
    for code in range(10):
        assert L.nfft_status_string(code)
    opt = pkg.Options()
    assert L.nfft_default_options(ctypes.byref(opt)) == 0
    assert opt.batch == 1 and opt.device == -1 and opt.check_nodes == 1 and opt.method == 0
    assert L.nfft_default_options(None) == 1  # NFFT_ERROR_INVALID_VALUE


def test_argument_validation_before_any_device_work(libpath):
    """Invalid arguments are rejected synchronously, before CUDA is touched."""
    L = pkg.lib()
    h = ctypes.c_void_p()
    N = (ctypes.c_int64 * 3)(16, 16, 16)
    nodes = (ctypes.c_double * 6)()
    create = L.nfft_plan_create
    assert create(None, 1, N, 2, nodes, 2.0, 2, 0, 1) == 1
    assert create(ctypes.byref(h), 4, N, 2, nodes, 2.0, 2, 0, 1) == 9   # D > 3 unsupported
    assert create(ctypes.byref(h), 0, N, 2, nodes, 2.0, 2, 0, 1) == 1
    assert create(ctypes.byref(h), 1, N, 0, nodes, 2.0, 2, 0, 1) == 1   # M < 1
    assert create(ctypes.byref(h), 1, N, 2, nodes, 1.0, 2, 0, 1) == 2   # sigma <= 1
    assert create(ctypes.byref(h), 1, N, 2, nodes, 2.0, 9, 0, 1) == 9   # m > 8
    N8 = (ctypes.c_int64 * 1)(8)
    assert create(ctypes.byref(h), 1, N8, 2, nodes, 2.0, 8, 0, 1) == 2  # 2m = 16 >= Ntilde = 16
    # N_d < 2 (odd N_d >= 3 are valid: PAPER.md:89)
    N1 = (ctypes.c_int64 * 1)(1)
    assert create(ctypes.byref(h), 1, N1, 2, nodes, 2.0, 2, 0, 1) == 2
    assert create(ctypes.byref(h), 1, N, 2, nodes, 2.0, 2, 5, 1) == 1   # unknown window
    # batch outside [1, 65535] (nfft_options.batch)
    opt = pkg.Options()
    L.nfft_default_options(ctypes.byref(opt))
    opt.batch = 65536
    assert L.nfft_plan_create_ex(ctypes.byref(h), 1, N, 2, nodes, 2.0, 2, 0, 1, ctypes.byref(opt)) == 9
    opt.batch = 0
    assert L.nfft_plan_create_ex(ctypes.byref(h), 1, N, 2, nodes, 2.0, 2, 0, 1, ctypes.byref(opt)) == 1
    assert L.nfft_forward(None, nodes, nodes) == 1
    assert L.nfft_precompute(None) == 1
