"""The branch-free correctly-rounded sqrt / reciprocal used inside the fused
pipeline kernels equal the IEEE intrinsics bit for bit (2^30 random doubles
over 80 binades each)."""

import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_fast_sqrt_rcp_bit_exact():
    from paper_2005_02704_b200 import _lib
    lib = _lib.lib()
    fn = lib.lseg_selftest_math
    fn.restype = C.c_int
    fn.argtypes = [C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p]
    bad = torch.zeros(2, dtype=torch.int64, device="cuda")
    for seed in (1, 2):
        _lib.check(fn(1 << 30, seed, C.c_void_p(bad.data_ptr()), _lib.stream_ptr()))
        torch.cuda.synchronize()
        assert bad.tolist() == [0, 0], f"sqrt / rcp mismatches: {bad.tolist()}"
