"""ctypes binding of liberx_probe.so (include/erx_probe.h): device probes and
tcgen05 self-tests.  Design evidence, not the ERX path: bench.py reads the
measured FFMA peak from here for the FFMA-bound kernels' roofline, and
tests/test_tc_selftest.py checks the descriptor layouts the exact-integer
kernels use.  No fallback: a missing library raises."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
PROBE_PATH = os.path.join(_HERE, "liberx_probe.so")
_probe = None

_vp, _dp = C.c_void_p, C.POINTER(C.c_double)
SIGNATURES = {
    "erx_probe_fp32_tflops": (C.c_int, [C.c_int, _vp, _dp, _dp]),
    "erx_probe_ffma2_tflops": (C.c_int, [C.c_int, _vp, _dp]),
    "erx_probe_stream": (C.c_int, [C.c_int, _vp, C.c_int, C.c_uint32, C.c_int, C.c_int, C.c_uint64, _dp]),
    "erx_tc_selftest": (C.c_int, [C.c_int, _vp, _vp, _vp, C.c_int, C.c_int, _vp]),
    "erx_tc_selftest_i8": (C.c_int, [C.c_int, _vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_int, _vp]),
}


def lib():
    global _probe
    if _probe is None:
        if not os.path.exists(PROBE_PATH):
            raise RuntimeError(f"{PROBE_PATH} not built (__graft_entry__.build())")
        L = C.CDLL(PROBE_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _probe = L
    return _probe


def _ok(st: int, what: str):
    if st:
        raise RuntimeError(f"{what}: status {st}")


def fp32_tflops(device: int = 0, stream: int = 0):
    """(register-form, constant-form) measured FFMA TFLOP/s of the device."""
    r, c = C.c_double(0), C.c_double(0)
    _ok(lib().erx_probe_fp32_tflops(device, stream or None, C.byref(r), C.byref(c)), "erx_probe_fp32_tflops")
    return float(r.value), float(c.value)


def ffma2_tflops(device: int = 0, stream: int = 0) -> float:
    t = C.c_double(0)
    _ok(lib().erx_probe_ffma2_tflops(device, stream or None, C.byref(t)), "erx_probe_ffma2_tflops")
    return float(t.value)


def stream_gbs(mode: int, chunk_bytes: int, stages: int, ctas_per_sm: int, nbytes: int, device: int = 0,
               stream: int = 0) -> float:
    g = C.c_double(0)
    _ok(lib().erx_probe_stream(device, stream or None, mode, chunk_bytes, stages, ctas_per_sm, nbytes, C.byref(g)),
        "erx_probe_stream")
    return float(g.value)
