"""CPU: the C-ABI library loads and exports every symbol include/ntc_b200.h
declares (no compute without a GPU); the product path refuses to run without
a device instead of falling back."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "ntc_b200.h")
LIB = os.path.join(ROOT, "paper_2109_09534_b200", "libntcb.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ntcb_[a-z0-9_]+)\s*\(", src)) - {"ntcb_observer_fn"})


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2109_09534_b200 import build
        build.build()
    return ctypes.CDLL(LIB)


def test_every_declared_symbol_is_exported(lib):
    names = declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_2109_09534_b200._lib import SIGNATURES
    assert sorted(SIGNATURES) == declared()


def test_host_helpers_match_reference_streams(lib, golden):
    lib.ntcb_sweep_stream_state.restype = ctypes.c_uint64
    lib.ntcb_sweep_stream_state.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int]
    lib.ntcb_rng_fork.restype = ctypes.c_uint64
    lib.ntcb_rng_fork.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    import oracle
    o = oracle.Oracle()
    for k in range(3):
        for m in range(4):
            assert lib.ntcb_sweep_stream_state(7, k, m) == o.sweep_state(7, k, m)
    assert lib.ntcb_rng_fork(42, 3) == o.fork(42, 3)


def test_no_silent_cpu_fallback(lib):
    """Without a CUDA device ntcb_create must fail loudly (NTCB_ECUDA/EINVAL)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    rc = lib.ntcb_create(0, ctypes.byref(h))
    assert rc != 0
    import paper_2109_09534_b200 as P
    with pytest.raises((P.CudaError, P.InvalidArgument)):
        P.Context(0)


def test_sources_are_sm100a_only():
    from paper_2109_09534_b200 import build
    assert build.ARCH == ["-gencode", "arch=compute_100a,code=sm_100a"]
    assert "-lineinfo" in build.FLAGS
