"""Helpers for the kind::f16 accumulator probe (tests/cuda/tc_probe.cu tc_bf16_acc) — test
infrastructure shared by tests/test_gpu_tcgen05.py and tools/acc_probe.py."""
import ctypes as C
import os

import numpy as np

SO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cuda", "libtcprobe.so")
_lib = None


def bf16_bits(a):
    """float32 -> bf16 bit patterns, round to nearest even."""
    b = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    r = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def bf16_val(a):
    """float32 rounded to the nearest bf16, as float32."""
    return (bf16_bits(a).astype(np.uint32) << 16).view(np.float32)


def f16_val(a):
    """float32 rounded to the nearest fp16 (round to nearest even), as float32."""
    return np.ascontiguousarray(a, np.float32).astype(np.float16).astype(np.float32)


def run_acc(A, B, Cinit=None, fp16=False):
    """D[128 x 32] = Cinit + A . B^T on the tensor core (A: 128 x K, B: 32 x K, values bf16-exact,
    or fp16-exact with fp16=True)."""
    global _lib
    if _lib is None:
        _lib = C.CDLL(SO)
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    assert A.shape[0] == 128 and B.shape[0] == 32 and A.shape[1] == B.shape[1]
    if fp16:
        assert np.array_equal(f16_val(A), A) and np.array_equal(f16_val(B), B), "operands must be fp16 values"
        ab, bb = A.astype(np.float16).view(np.uint16), B.astype(np.float16).view(np.uint16)
    else:
        ab, bb = bf16_bits(A), bf16_bits(B)
        assert np.array_equal(bf16_val(A), A) and np.array_equal(bf16_val(B), B), "operands must be bf16 values"
    D = np.zeros((128, 32), np.float32)
    has_c = Cinit is not None
    Cm = np.ascontiguousarray(Cinit if has_c else np.zeros((128, 32)), np.float32)
    u16 = C.POINTER(C.c_uint16)
    fp = C.POINTER(C.c_float)
    fn = _lib.tc_f16_acc if fp16 else _lib.tc_bf16_acc
    ab, bb = np.ascontiguousarray(ab), np.ascontiguousarray(bb)
    rc = fn(ab.ctypes.data_as(u16), bb.ctypes.data_as(u16), Cm.ctypes.data_as(fp), int(has_c),
                          A.shape[1], D.ctypes.data_as(fp))
    assert rc == 0, rc
    return D
