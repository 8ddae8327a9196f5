"""The C-ABI library loads and exports every symbol include/ks.h declares;
compute calls fail loudly (no CPU fallback) when no device is present."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ks.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ks_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(ks):
    L = ctypes.CDLL(ks.LIB_PATH)
    names = _declared()
    assert len(names) > 40
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # and the Python mirror binds every one of them
    assert set(names) <= set(ks._SIGS), set(names) - set(ks._SIGS)


def test_cpp_wrapper_header_compiles(tmp_path):
    # include/kronschro_gpu.hpp (the reference-signature wrappers) is self-contained
    src = tmp_path / "t.cpp"
    src.write_text('#include "kronschro_gpu.hpp"\nint main(){return 0;}\n')
    rc = os.system(f"g++ -std=c++17 -fsyntax-only -I{ROOT}/include {src}")
    assert rc == 0


def test_no_cpu_fallback(ks):
    if ks.device_count() > 0:
        pytest.skip("a device is present")
    prob = ks.SpaceTimeProblem.uniform(1, 2, 4, 4)
    with pytest.raises(ks.CudaError):
        ks.FDPreconditioner(prob)
    with pytest.raises(ks.CudaError):
        ks.assemble_system_operator(prob)


def test_error_codes(ks):
    with pytest.raises(ks.InvalidArgument):
        ks.SpaceTimeProblem.uniform(4, 2, 4, 4)
    with pytest.raises(ks.InvalidArgument):
        ks.SpaceTimeProblem.uniform(1, 2, 4, 4, T=-1.0)
    K = ks.KroneckerOperator([2, 2])
    with pytest.raises(ks.InvalidArgument):
        K.add_term(1.0, [ks.Banded(3, 1), None])  # factor size mismatch (test_tensorops.cpp:144-150)
    with pytest.raises(ks.InvalidArgument):
        K.add_term(1.0, [None])                    # wrong factor count
    with pytest.raises(ks.InvalidArgument):
        ks.KroneckerOperator([2, 0])                # CoeffTensor({2, 0}) throws
