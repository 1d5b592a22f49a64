"""Parity-gate metrics on the device, behind the C ABI
(erx_metrics_roc_auc / erx_metrics_top_k, csrc/k_metrics.cu).

Mirrors had::roc_curve's AUC (proj/include/hadkit/metrics.hpp:25-28) and the
pooled evaluation of evaluate_run (metrics.hpp:54-58): exact AUC with tied
scores grouped into one ROC step, MetricUndefinedError when a class is empty.
Arguments are device buffers: torch CUDA tensors (scores float32, labels /
select uint8 or bool) or raw device pointers with an explicit ``n``.
"""
import ctypes as C
from typing import Optional, Tuple

from . import _lib as L
from .detector import _raise


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _n(t, n):
    if n is not None:
        return int(n)
    return int(t.numel())


def _check_dtype(t, kinds, what):
    if t is None or isinstance(t, int):
        return
    name = str(t.dtype).replace("torch.", "")
    if name not in kinds:
        raise TypeError(f"{what}: dtype {name}, expected one of {kinds}")
    if not t.is_cuda or not t.is_contiguous():
        raise TypeError(f"{what}: a contiguous CUDA tensor is required")


def roc_auc(scores, labels, select=None, n: Optional[int] = None, stream: int = 0) -> float:
    """Exact ROC AUC of the selected device scores (fp32) against 0/1 labels."""
    _check_dtype(scores, ("float32",), "scores")
    _check_dtype(labels, ("uint8", "bool"), "labels")
    _check_dtype(select, ("uint8", "bool"), "select")
    auc = C.c_double(0.0)
    npos, nneg = C.c_uint64(0), C.c_uint64(0)
    st = L.lib().erx_metrics_roc_auc(_ptr(scores), _ptr(labels), _ptr(select), _n(scores, n), stream or None,
                                     C.byref(auc), C.byref(npos), C.byref(nneg))
    if st:
        _raise(st, f"roc_auc: npos={npos.value} nneg={nneg.value}")
    return auc.value


def top_k(scores, k: int, select=None, mask=None, n: Optional[int] = None, stream: int = 0) -> Tuple[object, float]:
    """Mask (uint8, 1 = among the k largest selected scores, ties to the lower index) and the cutoff."""
    _check_dtype(scores, ("float32",), "scores")
    _check_dtype(select, ("uint8", "bool"), "select")
    nn = _n(scores, n)
    if mask is None:
        import torch
        mask = torch.empty(nn, dtype=torch.uint8, device=scores.device)
    cut = C.c_float(0.0)
    st = L.lib().erx_metrics_top_k(_ptr(scores), _ptr(select), nn, int(k), stream or None, _ptr(mask),
                                   C.byref(cut))
    if st:
        _raise(st, f"top_k: k={k} n={nn}")
    return mask, cut.value
