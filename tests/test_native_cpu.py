"""CPU-side checks of the C-ABI library (no GPU needed, no compute calls).

The library must load, export every symbol include/ulysses_b200.h
declares, and reject bad arguments with the reference's error taxonomy
before touching a device.
"""

import ctypes
import os
import re
from fractions import Fraction

import pytest

from conftest import ROOT

from oracle import ulysses_oracle as O


def lib():
    from paper_2309_14509_b200 import _lib
    return _lib


def header_symbols():
    text = open(os.path.join(ROOT, "include", "ulysses_b200.h")).read()
    return sorted(set(re.findall(r"\b(ul_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_abi():
    L = lib().lib()
    assert L.ul_abi_version() == lib().ABI_VERSION == 2


def test_every_header_symbol_is_exported():
    L = lib().lib()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), f"{s} declared in include/ulysses_b200.h but not exported"
    assert sorted(lib().EXPORTS) == syms


def test_ulysses_volume_matches_oracle_and_costmodel():
    # costmodel.py:82-87 through the C-ABI vs the oracle restatement
    L = lib().lib()
    num, den = ctypes.c_int64(), ctypes.c_int64()
    for (n, b, d, p) in [(8, 1, 8, 4), (1024, 1, 512, 4), (65536, 1, 7168, 8), (8, 1, 8, 1)]:
        for conv, name in ((0, "exact"), (1, "paper_asymptotic")):
            assert L.ul_ulysses_volume(n, b, d, p, conv, ctypes.byref(num), ctypes.byref(den)) == 0
            assert Fraction(num.value, den.value) == O.ulysses_volume(n, b, d, p, name)


def test_attention_argument_errors_before_any_launch():
    from paper_2309_14509_b200 import errors
    L = lib().lib()
    # GQA divisibility
    st = L.ul_attn_fwd(None, None, None, None, None, 4, 1, 4, 3, 64, 1, 0, 0.1, None, None)
    assert errors.STATUS[st] is errors.DivisibilityError
    assert b"does not divide" in L.ul_last_error()
    # unsupported mask kind -> KernelError (kernels.py:43-52)
    st = L.ul_attn_fwd(None, None, None, None, None, 4, 1, 4, 4, 64, 1, 7, 0.1, None, None)
    assert errors.STATUS[st] is errors.KernelError
    # backward without LSE -> ForwardStateError (ulysses.py:198-207)
    p = ctypes.c_void_p(16)
    st = L.ul_attn_bwd(p, p, p, p, p, None, p, p, p, p, 1 << 20, 4, 1, 4, 4, 64, 1, 1, 0.1, 0, None)
    assert errors.STATUS[st] is errors.ForwardStateError
    # unknown per-call backward flags -> ValueError (UL_ERR_ARG), before any launch
    st = L.ul_attn_bwd(p, p, p, p, p, p, p, p, p, p, 1 << 20, 4, 1, 4, 4, 64, 1, 1, 0.1, 4, None)
    assert st == -8 and b"flags" in L.ul_last_error()


def test_all_to_all_argument_errors_before_any_launch():
    from paper_2309_14509_b200 import errors
    L = lib().lib()
    shapes = (ctypes.c_int64 * 4)(3, 2, 0, 0)
    ptrs = (ctypes.c_void_p * 1)(16)
    # too many fused tensors
    st = L.ul_all_to_all(None, 9, ptrs, ptrs, shapes, 2, 0, 0, 1, 0, None)
    assert errors.STATUS[st] is ValueError
    # axis out of range
    st = L.ul_all_to_all(None, 1, ptrs, ptrs, shapes, 2, 0, 2, 1, 0, None)
    assert errors.STATUS[st] is ValueError


def test_slot_bytes_geometry():
    L = lib().lib()
    shapes = (ctypes.c_int64 * 12)(64, 1, 32, 128, 64, 1, 8, 128, 64, 1, 8, 128)
    need = L.ul_all_to_all_slot_bytes(3, shapes, 4, 1, 2, 0, 8)
    # outputs (512, 1, 4|1|1, 128) bf16 each, 256-aligned
    assert need == 512 * 128 * 2 * (4 + 1 + 1)


def test_python_a2a_shape_rules_match_oracle():
    import numpy as np
    from paper_2309_14509_b200 import ShardError, a2a_out_shape
    for shape, p, s, c in [((4, 1, 8, 16), 4, 2, 0), ((32, 2, 2, 4), 8, 0, 2), ((8, 2, 8), 4, 0, 1)]:
        outs = O.all_to_all([np.zeros(shape)] * p, s, c)
        assert a2a_out_shape(shape, p, s, c) == outs[0].shape
    with pytest.raises(ShardError):
        a2a_out_shape((3, 2), 2, 0, 1)
