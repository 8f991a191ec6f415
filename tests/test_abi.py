"""CPU checks of the C-ABI boundary: the library builds, loads without a GPU and
exports every entry point include/fabf.h declares; the Python binding mirrors
them; the product package never imports the oracle."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fabf.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fabf_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1811_02308_b200 import build

    return build.build()


def test_header_declares_the_north_star_calls():
    names = _declared_functions()
    for n in ("fabf_plan", "fabf_filter", "fabf_destroy", "fabf_bounds", "fabf_filter_diag",
              "fabf_filter_host", "fabf_status_string", "fabf_last_error_message", "fabf_version"):
        assert n in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for name in _declared_functions():
        assert hasattr(lib, name), name


def test_library_is_sm100a_only(libpath):
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath],
                         capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, out


def test_status_strings_and_version(libpath):
    import paper_1811_02308_b200 as fb

    L = fb.lib()
    assert L.fabf_version() == 100
    for code, name in [(0, b"FABF_OK"), (1, b"FABF_ERR_INVALID_ARGUMENT"), (2, b"FABF_ERR_UNSUPPORTED"),
                       (3, b"FABF_ERR_CUDA"), (4, b"FABF_ERR_OUT_OF_MEMORY")]:
        assert L.fabf_status_string(code) == name


def test_plan_argument_errors_without_gpu(libpath):
    import paper_1811_02308_b200 as fb

    L = fb.lib()
    h = ctypes.c_void_p()
    assert L.fabf_plan(None, 1, 8, 8, 0) == 1
    assert L.fabf_plan(ctypes.byref(h), 0, 8, 8, 0) == 1
    assert L.fabf_plan(ctypes.byref(h), 1, 8, 8, 0x80) == 1
    assert b"flag" in L.fabf_last_error_message()
    assert L.fabf_destroy(None) == 0
    # NULL plan handle on the compute entry points is an argument error, not a crash
    assert L.fabf_filter(None, None, None, None, 1, 2, None, None) == 1
    assert L.fabf_bounds(None, None, 1, None, None, None) == 1


def test_no_cpu_fallback_on_a_cpu_box(libpath):
    """Without a GPU the plan fails loudly (CUDA error), it never computes."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1811_02308_b200 as fb

    with pytest.raises(fb.FabfError):
        fb.Plan(1, 16, 16)


def test_product_never_imports_oracle():
    """Only tests/, __graft_entry__.smoke() and bench.py may touch oracle/: the
    package and the tools/ drivers never import, link or run it."""
    for pkg in (os.path.join(ROOT, "paper_1811_02308_b200"), os.path.join(ROOT, "tools")):
      for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp", ".sh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "fabf_oracle" not in txt and "liboracle" not in txt, f


def test_binding_host_buffers_checked_without_gpu():
    """The binding refuses host buffers that are not float32 or do not hold the
    plan's pixel count (int32 would otherwise be reinterpreted as float)."""
    import numpy as np

    from paper_1811_02308_b200 import fabf

    class _P:
        shape = (1, 8, 8)

    ok = np.zeros((1, 8, 8), np.float32)
    assert fabf._host_ptr(ok, "img", _P()).value == ok.ctypes.data
    for bad in (ok.astype(np.int32), ok.astype(np.float64), np.zeros((1, 8, 4), np.float32),
                np.zeros((1, 8, 16), np.float32)[:, :, ::2]):
        with pytest.raises(fabf.FabfError):
            fabf._host_ptr(bad, "img", _P())


def test_binding_constants_match_header():
    """Every FABF_FLAG_* / FABF_CODE_* of include/fabf.h is exported by the
    package with the same value (the binding hard-codes them)."""
    import paper_1811_02308_b200 as fb

    src = open(HEADER).read()
    found = re.findall(r"#define\s+FABF_((?:FLAG|CODE)_[A-Z_]+)\s+(0x[0-9a-fA-F]+)u?", src)
    assert found
    for name, val in found:
        assert getattr(fb, name) == int(val, 16), name
