"""The drop-in boundary loads and exports every symbol include/eig33_cuda.h
declares; argument errors come back as status codes (no GPU needed)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2511_00292_b200 as eig
from tests import _util as U

HEADER = os.path.join(U.ROOT, "include", "eig33_cuda.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|long long)\s+(eig33\w*)\s*\(", src, flags=re.M)))


def test_header_matches_python_binding_table():
    assert _declared() == sorted(eig.C_ABI_SYMBOLS)


def test_library_exports_every_declared_symbol():
    L = eig.lib()
    for name in _declared():
        assert hasattr(L, name), name
    assert L.eig33cu_version() >> 16 == 1


def test_bad_arguments_return_status_without_touching_the_gpu():
    L = eig.lib()
    assert L.eig33cu_eigvals(None, 5, None, None, None, None) == eig.EIG33_EINVAL
    assert b"null" in L.eig33cu_last_error()
    assert L.eig33cu_invariants(None, 0, None, None) == eig.EIG33_OK  # empty batch
    assert L.eig33cu_generate(9, 0, 0, 4, ctypes.c_void_p(16), None) == eig.EIG33_EINVAL


def test_cxx_header_compiles():
    # include/eig33/batch.hpp: the C++ overloads with the reference's names
    import subprocess
    src = os.path.join(U.ROOT, "tests", "cpp", "batch_api_check.cpp")
    out = "/tmp/eig33_batch_api_check.o"
    r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-I", os.path.join(U.ROOT, "include"), src],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.parametrize("shape", [(4, 2, 2), (9,), (3, 4), (2, 3, 3, 1)])
def test_shape_validation_mirrors_reference_to_mat(shape):
    if shape == (9,):
        eig._records_np(np.zeros(shape))  # a single flat record is accepted
        return
    with pytest.raises(ValueError):
        eig._records_np(np.zeros(shape))


def test_entry_dtype_rules():
    """Real numeric host input is converted to float64 (the reference binding
    takes Python floats); complex, string and object input raise ValueError."""
    assert eig._records_np(np.arange(18, dtype=np.int32).reshape(2, 3, 3)).dtype == np.float64
    assert eig._records_np(np.ones((1, 9), np.float32)).dtype == np.float64
    for bad in (np.zeros((2, 3, 3), complex), np.array([["a"] * 9]), np.array([[None] * 9])):
        with pytest.raises(ValueError):
            eig._records_np(bad)


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"), reason="reference headers absent")
def test_cxx_header_compiles_against_reference_types():
    """Drop-in: with the reference's own headers on the include path, batch.hpp
    adds its overloads to the reference's Mat3 / InvariantSet / EigenTriple."""
    import subprocess
    src = os.path.join(U.ROOT, "tests", "cpp", "batch_api_check.cpp")
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(U.ROOT, "include"),
                        "-I", "/root/reference/proj/include", src], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
