"""HADC cube / mask files ([MODULE] io) over
the C ABI (csrc/hadc.cpp): read_cube / write_cube / read_mask / write_mask
with the reference's validation (bad magic, truncated payload, zero sizes,
unsupported dtype, mask values other than 0/1 -> FormatError, kind data,
carrying the file and byte offset; failing to open / read -> IoError), plus a reader that streams line ranges into host memory or, through
pinned double-buffered staging, straight into device memory for the engine.
"""
import ctypes as C
import re
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .detector import FormatError, _raise


def _fail(st: int, msg: str, path: str):
    """ERX_ERR_DATA from the reader is had::FormatError (errors.hpp:67-75): path + byte offset."""
    if st == L.ERX_ERR_DATA:
        m = re.search(r"at offset (\d+)", msg)
        raise FormatError(str(path), int(m.group(1)) if m else -1, msg)
    _raise(st, msg)

DTYPE_F32 = 1
DTYPE_U8 = 2


@dataclass
class CubeHeader:
    version: int
    lines: int
    pixels: int
    bands: int
    dtype: int
    layout: int
    name: str


class HadcReader:
    """An open HADC file: header fields plus line-range reads."""

    def __init__(self, path: str):
        self._h = C.c_void_p()
        info = L.HadcInfoC()
        self.path = str(path)
        st = L.lib().erx_hadc_open(str(path).encode(), C.byref(self._h), C.byref(info))
        if st:
            _fail(st, L.lib().erx_hadc_last_error(None).decode(errors="replace"), self.path)
        self.header = CubeHeader(info.version, info.lines, info.pixels, info.bands, info.dtype, info.layout,
                                 info.name.decode("utf-8", errors="replace"))

    def _check(self, st):
        if st:
            _fail(st, L.lib().erx_hadc_last_error(self._h).decode(errors="replace"), self.path)

    @property
    def np_dtype(self):
        return np.float32 if self.header.dtype == DTYPE_F32 else np.uint8

    def read(self, first: int = 0, n: int = None) -> np.ndarray:
        h = self.header
        n = h.lines - first if n is None else n
        out = np.empty((n, h.pixels, h.bands), self.np_dtype)
        self._check(L.lib().erx_hadc_read(self._h, first, n, out.ctypes.data))
        return out

    def read_into(self, first: int, n: int, host_ptr: int):
        """Lines into caller memory (e.g. an erx_host_alloc pinned buffer for erx_push_host)."""
        self._check(L.lib().erx_hadc_read(self._h, first, n, host_ptr))

    def read_device(self, first: int, n: int, out=None, stream: int = 0):
        """Lines into device memory (a torch CUDA tensor, allocated when `out` is None)."""
        h = self.header
        if out is None:
            import torch
            out = torch.empty((n, h.pixels, h.bands),
                              dtype=torch.float32 if h.dtype == DTYPE_F32 else torch.uint8, device="cuda")
        self._check(L.lib().erx_hadc_read_device(self._h, first, n, out.data_ptr(), stream or None))
        return out

    def close(self):
        if self._h:
            L.lib().erx_hadc_close(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def write_cube(path: str, cube: np.ndarray, name: str = ""):
    """write_cube: fp32 [lines][pixels][bands]."""
    a = np.ascontiguousarray(cube, np.float32)
    if a.ndim != 3:
        raise ValueError("cube must be [lines][pixels][bands]")
    st = L.lib().erx_hadc_write(str(path).encode(), name.encode(), a.shape[0], a.shape[1], a.shape[2], DTYPE_F32,
                                a.ctypes.data)
    if st:
        _raise(st, f"write_cube {path}: status {st}")


def write_mask(path: str, mask: np.ndarray, name: str = ""):
    """write_mask: u8 0/1 [lines][pixels] (stored with bands = 1)."""
    a = np.ascontiguousarray(mask, np.uint8)
    if a.ndim != 2:
        raise ValueError("mask must be [lines][pixels]")
    st = L.lib().erx_hadc_write(str(path).encode(), name.encode(), a.shape[0], a.shape[1], 1, DTYPE_U8,
                                a.ctypes.data)
    if st:
        _raise(st, f"write_mask {path}: status {st}")


def read_cube(path: str):
    with HadcReader(path) as r:
        if r.header.dtype != DTYPE_F32:
            raise FormatError(str(path), 18, f"{path}: not a cube (dtype {r.header.dtype})")
        return r.header, r.read()


def read_mask(path: str):
    with HadcReader(path) as r:
        if r.header.dtype != DTYPE_U8 or r.header.bands != 1:
            raise FormatError(str(path), 14, f"{path}: not a mask (dtype {r.header.dtype}, bands {r.header.bands})")
        return r.header, r.read()[:, :, 0]
