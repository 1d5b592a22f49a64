"""ctypes binding of liberx_b200.so (include/erx_b200.h, include/erx_datagen.h).

The shared library is built in-tree by `python -m paper_2408_14947_b200.build`
(or __graft_entry__.build()).  There is no fallback: if the library is
missing or the CUDA device is unusable, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ERX_B200_LIB", os.path.join(_HERE, "liberx_b200.so"))  # override: A/B builds

ERX_OK = 0
ERX_ERR_CONFIG = 2
ERX_ERR_DATA = 3
ERX_ERR_METRIC = 4
ERX_ERR_NUMERIC = 5
ERX_ERR_IO = 6
ERX_ERR_DEVICE = 16
ERX_ERR_STATE = 17
NUM_KERNELS = 6
KERNEL_NAMES = ("stats", "scan", "factor", "score", "normalize", "fixup")
OPT_FACTOR_PRECISION = 1
OPT_STATS_TENSOR = 2
OPT_HOST_GROUPS = 3
OPT_ASYNC_HOST = 4
OPT_FACTOR_THREADS = 5
OPT_GRAPHS = 6
OPT_DEVICE_GROUPS = 7
OPT_STATS_SPLIT = 8
OPT_STATS_ONEPASS = 9
OPT_STATS_REDONE = 10


class ErxConfigC(C.Structure):
    _fields_ = [
        ("dims", C.c_int32),
        ("alpha", C.c_double),
        ("buffer_len", C.c_uint32),
        ("epsilon", C.c_double),
        ("seed", C.c_uint64),
        ("no_srp", C.c_int32),
        ("use_incremental", C.c_int32),
    ]


class GenSpecC(C.Structure):
    _fields_ = [
        ("lines", C.c_uint32),
        ("pixels", C.c_uint32),
        ("bands", C.c_uint32),
        ("n_factors", C.c_uint32),
        ("loading_sd", C.c_double),
        ("noise_sd", C.c_double),
        ("base_kind", C.c_int32),
        ("drift", C.c_double),
        ("n_scene_changes", C.c_uint32),
        ("scene_change_line", C.c_int64 * 4),
        ("anomaly_frac", C.c_double),
        ("anomaly_kind", C.c_int32),
        ("offset_sd", C.c_double),
        ("mix_lo", C.c_double),
        ("mix_hi", C.c_double),
        ("seed", C.c_uint64),
    ]


class HadcInfoC(C.Structure):
    _fields_ = [
        ("version", C.c_uint16),
        ("lines", C.c_uint32),
        ("pixels", C.c_uint32),
        ("bands", C.c_uint32),
        ("dtype", C.c_uint8),
        ("layout", C.c_uint8),
        ("name_len", C.c_uint16),
        ("name", C.c_char * 256),
    ]


# name -> (restype, argtypes)
_vp, _dp, _fp, _u8p, _i64p, _u64p = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_float), \
    C.POINTER(C.c_uint8), C.POINTER(C.c_int64), C.POINTER(C.c_uint64)
SIGNATURES = {
    "erx_config_default": (None, [C.POINTER(ErxConfigC)]),
    "erx_config_validate": (C.c_int, [C.POINTER(ErxConfigC), C.c_uint32, C.c_char_p, C.c_size_t]),
    "erx_generate_srp": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, _dp]),
    "erx_create": (C.c_int, [C.POINTER(ErxConfigC), C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                             C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]),
    "erx_destroy": (None, [_vp]),
    "erx_last_error": (C.c_char_p, [_vp]),
    "erx_last_pivot": (C.c_int, [_vp]),
    "erx_dims": (C.c_int, [_vp]),
    "erx_streams": (C.c_uint32, [_vp]),
    "erx_window": (C.c_uint32, [_vp]),
    "erx_push_host": (C.c_int, [_vp, C.c_int64, C.c_uint32, C.c_uint32, C.c_uint32, _fp]),
    "erx_finish": (C.c_int, [_vp]),
    "erx_ready": (C.c_uint32, [_vp]),
    "erx_next_pixels": (C.c_uint32, [_vp]),
    "erx_pop": (C.c_int, [_vp, C.c_uint32, _i64p, _u8p, _dp, _dp]),
    "erx_run_device": (C.c_int, [_vp, C.c_int64, C.c_uint32, C.c_uint32, _vp, _vp, _vp]),
    "erx_advance_device": (C.c_int, [_vp, C.c_int64, C.c_uint32, C.c_uint32, _vp]),
    "erx_sync": (C.c_int, [_vp]),
    "erx_cuda_stream": (C.c_void_p, [_vp]),
    "erx_get_state": (C.c_int, [_vp, C.c_uint32, _dp, _dp, _i64p, _i64p, C.POINTER(C.c_int)]),
    "erx_get_weights": (C.c_int, [_vp, _dp]),
    "erx_set_state": (C.c_int, [_vp, C.c_uint32, _dp, _dp, C.c_int64, C.c_int64]),
    "erx_launch_count": (C.c_uint64, [_vp]),
    "erx_set_option": (C.c_int, [_vp, C.c_int, C.c_int64]),
    "erx_get_option": (C.c_int64, [_vp, C.c_int]),
    "erx_set_profiling": (C.c_int, [_vp, C.c_int]),
    "erx_kernel_times": (C.c_int, [_vp, _dp, _u64p]),
    "erx_rescued_lines": (C.c_int64, [_vp]),
    "erx_metrics_roc_auc": (C.c_int, [_vp, _vp, _vp, C.c_size_t, _vp, _dp, _u64p, _u64p]),
    "erx_metrics_top_k": (C.c_int, [_vp, _vp, C.c_size_t, C.c_size_t, _vp, _vp, _fp]),
    "erx_hadc_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(HadcInfoC)]),
    "erx_hadc_last_error": (C.c_char_p, [_vp]),
    "erx_hadc_read": (C.c_int, [_vp, C.c_uint32, C.c_uint32, _vp]),
    "erx_hadc_read_device": (C.c_int, [_vp, C.c_uint32, C.c_uint32, _vp, _vp]),
    "erx_hadc_close": (None, [_vp]),
    "erx_hadc_write": (C.c_int, [C.c_char_p, C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, _vp]),
    "erx_event_record": (C.c_int, [_vp, C.c_int]),
    "erx_event_elapsed_ms": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "erx_host_alloc": (C.c_void_p, [C.c_size_t]),
    "erx_host_free": (None, [_vp]),
    "erx_device_alloc": (C.c_void_p, [C.c_int, C.c_size_t]),
    "erx_device_free": (None, [_vp]),
    "erx_copy": (C.c_int, [_vp, _vp, C.c_size_t, C.c_int, _vp]),
    "erx_gen_preset": (C.c_int, [C.c_int, C.c_uint32, C.POINTER(GenSpecC)]),
    "erx_gen_lines": (C.c_int, [C.POINTER(GenSpecC), C.c_uint32, C.c_uint32, _fp, _u8p, C.c_int]),
    "erx_gen_lines_device": (C.c_int, [C.POINTER(GenSpecC), C.c_uint32, C.c_uint32, _vp, _vp, _vp]),
    "erx_gen_scene_changes": (C.c_int, [C.POINTER(GenSpecC), _i64p]),
    "erx_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "erx_rng_probe": (None, [C.c_uint64, C.c_int, C.c_uint32, _u64p, _dp]),
}

_lib = None


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load liberx_b200.so (raises LibraryMissing: no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(nvcc, sm_100a). The ERX path has no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
