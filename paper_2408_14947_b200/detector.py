"""Python mirror of the reference detector interface, backed by liberx_b200.so.

Mirrors, name for name, the C++ contract in proj/include/hadkit/:
  ErxConfig        erx.hpp:14-24     (validate() -> ConfigError)
  ErxState         erx.hpp:27-34
  SpectralLine     cube.hpp:48-55    (index, pixels, bands, data p x b fp32)
  ScoredLine       cube.hpp:76-82    (index, raw, norm, decisions, warmup)
  LineDetector     detector.hpp:15-27 (process / finish / name / emits_normalized_scores)
  ErxDetector      erx.hpp:56-71     (constructed with (cfg, bands))
  apply_threshold  erx.hpp:46-47
  error types      errors.hpp:12-79 (same ErrorKind codes and exit codes)

Every score comes from the sm_100a kernels behind the C ABI; nothing here
computes a score on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L


# ---------------------------------------------------------------- errors (errors.hpp:12-79)
class Error(RuntimeError):
    kind = 0

    def exit_code(self) -> int:  # errors.hpp:27-33
        return {2: 2, 4: 4}.get(self.kind, 3)


class ConfigError(Error):
    kind = 2


class DataError(Error):
    kind = 3


class MetricUndefinedError(Error):
    kind = 4


class FactorizationError(Error):
    kind = 5

    def __init__(self, pivot: int, msg: str):
        super().__init__(msg)
        self.pivot = pivot


class IoError(Error):
    kind = 6


class FormatError(DataError):
    """Malformed or truncated file (errors.hpp:67-75): kind data, with the file and byte offset."""

    def __init__(self, path: str, offset: int, msg: str):
        super().__init__(f"{msg} (file '{path}', offset {offset})")
        self.path = path
        self.offset = offset


class DeviceError(Error):
    """CUDA failure inside the engine (no reference analogue)."""
    kind = 16


def _raise(code: int, msg: str, pivot: int = -1):
    if code == L.ERX_ERR_CONFIG:
        raise ConfigError(msg)
    if code == L.ERX_ERR_DATA:
        raise DataError(msg)
    if code == L.ERX_ERR_METRIC:
        raise MetricUndefinedError(msg)
    if code == L.ERX_ERR_NUMERIC:
        raise FactorizationError(pivot, msg)
    if code == L.ERX_ERR_IO:
        raise IoError(msg)
    raise DeviceError(f"[{code}] {msg}")


# ---------------------------------------------------------------- data model (cube.hpp)
@dataclass
class SpectralLine:
    index: int
    data: np.ndarray  # p x b, fp32, row-major (band fastest)

    @property
    def pixels(self) -> int:
        return int(self.data.shape[0])

    @property
    def bands(self) -> int:
        return int(self.data.shape[1])


@dataclass
class ScoredLine:
    index: int
    raw: np.ndarray
    norm: np.ndarray
    decisions: Optional[np.ndarray] = None
    warmup: bool = False


@dataclass
class ErxConfig:
    dims: int = 5
    alpha: float = 0.1
    buffer_len: int = 99
    epsilon: float = 1e-5
    seed: int = 0
    no_srp: bool = False
    use_incremental: bool = False

    def c(self) -> L.ErxConfigC:
        return L.ErxConfigC(self.dims, self.alpha, self.buffer_len, self.epsilon, self.seed, int(self.no_srp),
                            int(self.use_incremental))

    def validate(self, bands: int = 1 << 30) -> None:
        msg = C.create_string_buffer(256)
        c = self.c()
        st = L.lib().erx_config_validate(C.byref(c), bands, msg, 256)
        if st:
            _raise(st, msg.value.decode())


@dataclass
class ErxState:
    weights: Optional[np.ndarray]
    mu: np.ndarray
    cov: np.ndarray
    lines_seen: int = 0
    welford_n: int = 0
    initialized: bool = False


def apply_threshold(norm_scores, tau: float) -> np.ndarray:
    """erx::apply_threshold (erx.hpp:46-47): y_i = 1 iff norm_i >= tau."""
    return (np.asarray(norm_scores) >= tau).astype(np.uint8)


def generate_srp(bands: int, dims: int, seed: int) -> np.ndarray:
    """generate_srp (projection.hpp:26), host-side restatement in liberx_b200.so."""
    w = np.zeros((bands, dims), np.float64)
    st = L.lib().erx_generate_srp(bands, dims, seed, w.ctypes.data_as(C.POINTER(C.c_double)))
    if st:
        _raise(st, "generate_srp: bands and dims must be >= 1")
    return w


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


# ---------------------------------------------------------------- the engine
class Engine:
    """S independent ERX streams advanced in lock-step on one GPU (C ABI erx_engine)."""

    def __init__(self, cfg: ErxConfig, bands: int, n_streams: int = 1, window_lines: int = 32, device: int = 0):
        self._lib = L.lib()
        self.cfg = cfg
        self.bands = bands
        self.n_streams = n_streams
        self.window = window_lines
        h = C.c_void_p()
        msg = C.create_string_buffer(512)
        c = cfg.c()
        st = self._lib.erx_create(C.byref(c), bands, n_streams, window_lines, device, C.byref(h), msg, 512)
        if st:
            _raise(st, msg.value.decode())
        self._h = h
        self.dims = self._lib.erx_dims(h)
        self.pixels = None

    def close(self):
        if getattr(self, "_h", None):
            self._lib.erx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int):
        if st:
            _raise(st, self._lib.erx_last_error(self._h).decode(), self._lib.erx_last_pivot(self._h))

    # drop-in host path
    def push(self, lines: np.ndarray, first_index: int):
        """lines: [S][n][P][B] fp32 host array."""
        x = np.ascontiguousarray(lines, np.float32)
        if x.ndim != 4 or x.shape[0] != self.n_streams:
            raise DataError("lines must be [n_streams][n_lines][pixels][bands]")
        S, n, P, B = x.shape
        self.pixels = P
        self._check(self._lib.erx_push_host(self._h, first_index, n, P, B, _p(x, C.c_float)))

    def finish(self):
        self._check(self._lib.erx_finish(self._h))

    def ready(self) -> int:
        return int(self._lib.erx_ready(self._h))

    def pop(self, max_lines: Optional[int] = None, out=None):
        """Pop the leading ready lines: (index[n], warmup[n], raw[S][n][P], norm[S][n][P]) fp64.

        `out` = (raw, norm) preallocated C-contiguous fp64 arrays of at least n x P
        per stream reuses caller memory (views of the first n lines are returned)."""
        n = self.ready() if max_lines is None else min(max_lines, self.ready())
        P = int(self._lib.erx_next_pixels(self._h))
        idx = np.zeros(n, np.int64)
        wu = np.zeros(n, np.uint8)
        if out is not None:
            raw_o, norm_o = out
            need = self.n_streams * n * P
            if raw_o.dtype != np.float64 or norm_o.dtype != np.float64 or raw_o.size < need or norm_o.size < need \
                    or not raw_o.flags.c_contiguous or not norm_o.flags.c_contiguous:
                raise DataError("pop(out=...) needs two C-contiguous float64 arrays of >= S*n*P elements")
            raw = raw_o.reshape(-1)[:need].reshape(self.n_streams, n, P)
            norm = norm_o.reshape(-1)[:need].reshape(self.n_streams, n, P)
        else:
            raw = np.empty((self.n_streams, n, P))
            norm = np.empty((self.n_streams, n, P))
        got = self._lib.erx_pop(self._h, n, _p(idx, C.c_int64), _p(wu, C.c_uint8), _p(raw, C.c_double),
                                _p(norm, C.c_double))
        if got < 0:
            self._check(-got)
        return idx, wu.astype(bool), raw, norm

    # device-resident path
    def run_device(self, d_lines: int, n_lines: int, pixels: int, d_raw: int, d_norm: int, first_index: int = 0):
        self.pixels = pixels
        self._check(self._lib.erx_run_device(self._h, first_index, n_lines, pixels, C.c_void_p(d_lines),
                                             C.c_void_p(d_raw), C.c_void_p(d_norm)))

    def advance_device(self, d_lines: int, n_lines: int, pixels: int, first_index: int = 0):
        """Background update only (statistics + scan, no scores): erx_advance_device."""
        self.pixels = pixels
        self._check(self._lib.erx_advance_device(self._h, first_index, n_lines, pixels, C.c_void_p(d_lines)))

    def sync(self):
        self._check(self._lib.erx_sync(self._h))

    def state(self, stream: int = 0) -> ErxState:
        d = self.dims
        mu = np.zeros(d)
        cov = np.zeros((d, d))
        ls, wn, ini = C.c_int64(0), C.c_int64(0), C.c_int(0)
        self._check(self._lib.erx_get_state(self._h, stream, _p(mu, C.c_double), _p(cov, C.c_double), C.byref(ls),
                                            C.byref(wn), C.byref(ini)))
        w = None
        if not self.cfg.no_srp:
            w = np.zeros((self.bands, d))
            self._lib.erx_get_weights(self._h, _p(w, C.c_double))
        return ErxState(w, mu, cov, ls.value, wn.value, bool(ini.value))

    def set_state(self, stream: int, mu, cov, lines_seen: int, welford_n: int = 0):
        mu = np.ascontiguousarray(mu, np.float64)
        cov = np.ascontiguousarray(cov, np.float64)
        self._check(self._lib.erx_set_state(self._h, stream, _p(mu, C.c_double), _p(cov, C.c_double), lines_seen,
                                            welford_n))

    def set_factor_precision(self, bits: int):
        """0 auto, 32 or 64 (see ERX_OPT_FACTOR_PRECISION in include/erx_b200.h)."""
        self._check(self._lib.erx_set_option(self._h, L.OPT_FACTOR_PRECISION, bits))

    def set_stats_onepass(self, headroom: int):
        """Headroom of the one-pass statistics' predicted range, 0 for the two-pass kernels (ERX_OPT_STATS_ONEPASS)."""
        self._check(self._lib.erx_set_option(self._h, L.OPT_STATS_ONEPASS, int(headroom)))

    def stats_redone_lines(self) -> int:
        """Lines the one-pass statistics handed to the exact two-pass kernel so far (ERX_OPT_STATS_REDONE)."""
        return int(self._lib.erx_get_option(self._h, L.OPT_STATS_REDONE))

    def set_stats_split(self, ring1: int):
        """Pass-1 stages of the split statistics kernel, 0 for the single-role kernel (ERX_OPT_STATS_SPLIT)."""
        self._check(self._lib.erx_set_option(self._h, L.OPT_STATS_SPLIT, int(ring1)))

    def set_device_groups(self, groups: int):
        """Device stream groups per window: 0 auto, 1 or 2 (ERX_OPT_DEVICE_GROUPS)."""
        self._check(self._lib.erx_set_option(self._h, L.OPT_DEVICE_GROUPS, int(groups)))

    def set_factor_threads(self, threads: int):
        """Threads per line of the blocked fp32 factor: 0 auto, 64, 128 or 256 (ERX_OPT_FACTOR_THREADS)."""
        self._check(self._lib.erx_set_option(self._h, L.OPT_FACTOR_THREADS, int(threads)))

    def set_stats_tensor(self, kind: int):
        """Line-statistics kernel: 0 FFMA, 1 tcgen05 bf16x3, 2 tcgen05 exact int8 (ERX_OPT_STATS_TENSOR)."""
        self._check(self._lib.erx_set_option(self._h, L.OPT_STATS_TENSOR, int(kind)))

    def set_host_groups(self, groups: int):
        """Stream groups per host window (0 auto; see ERX_OPT_HOST_GROUPS)."""
        self._check(self._lib.erx_set_option(self._h, L.OPT_HOST_GROUPS, int(groups)))

    def set_graphs(self, on: bool):
        """Replay erx_run_device windows as CUDA graphs (ERX_OPT_GRAPHS, default on)."""
        self._check(self._lib.erx_set_option(self._h, L.OPT_GRAPHS, int(bool(on))))

    def set_async_host(self, on: bool):
        """Pipelined host path (ERX_OPT_ASYNC_HOST): push returns once the input is on the device;
        windows are harvested by ready / pop / finish."""
        self._check(self._lib.erx_set_option(self._h, L.OPT_ASYNC_HOST, 1 if on else 0))

    def stats_tensor(self) -> int:
        """Line-statistics kernel in use (0 FFMA, 1 bf16x3, 2 exact int8)."""
        return int(self._lib.erx_get_option(self._h, L.OPT_STATS_TENSOR))

    def factor_precision(self) -> int:
        return int(self._lib.erx_get_option(self._h, L.OPT_FACTOR_PRECISION))

    # instrumentation
    def launch_count(self) -> int:
        return int(self._lib.erx_launch_count(self._h))

    def set_profiling(self, on: bool):
        self._lib.erx_set_profiling(self._h, int(on))

    def rescued_lines(self) -> int:
        """Lines redone by the fp64 rescue kernel so far (erx_rescued_lines)."""
        return int(self._lib.erx_rescued_lines(self._h))

    def kernel_times(self):
        ms = np.zeros(L.NUM_KERNELS)
        n = np.zeros(L.NUM_KERNELS, np.uint64)
        self._lib.erx_kernel_times(self._h, _p(ms, C.c_double), _p(n, C.c_uint64))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(L.KERNEL_NAMES)}

    def event_record(self, slot: int):
        self._check(self._lib.erx_event_record(self._h, slot))

    def event_elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float(0)
        self._check(self._lib.erx_event_elapsed_ms(self._h, a, b, C.byref(ms)))
        return float(ms.value)

    @property
    def cuda_stream(self) -> int:
        return int(self._lib.erx_cuda_stream(self._h) or 0)


class LineDetector:
    """detector.hpp:15-27."""

    def process(self, line: SpectralLine, out: List[ScoredLine]) -> None:
        raise NotImplementedError

    def finish(self, out: List[ScoredLine]) -> None:
        return None

    def name(self) -> str:
        raise NotImplementedError

    def emits_normalized_scores(self) -> bool:
        return False


class ErxDetector(LineDetector):
    """had::ErxDetector (erx.hpp:56-71) on the B200.

    `window_lines` is the pipelining lag allowed by detector.hpp:11-14: up to
    that many lines are scored per device pass; finish() flushes the rest.
    window_lines=1 scores every line before process() returns.
    """

    def __init__(self, cfg: ErxConfig, bands: int, window_lines: int = 32, device: int = 0):
        self._cfg = cfg
        self._bands = bands
        self._eng = Engine(cfg, bands, 1, window_lines, device)

    def _drain(self, out: List[ScoredLine]):
        while self._eng.ready():
            idx, wu, raw, norm = self._eng.pop()
            for k in range(idx.size):
                out.append(ScoredLine(int(idx[k]), raw[0, k].copy(), norm[0, k].copy(), None, bool(wu[k])))

    def process(self, line: SpectralLine, out: List[ScoredLine]) -> None:
        data = np.asarray(line.data, np.float32)
        if data.ndim != 2:
            raise DataError("SpectralLine.data must be p x b")
        try:
            self._eng.push(data[None, None], int(line.index))
        finally:
            self._drain(out)

    def finish(self, out: List[ScoredLine]) -> None:
        try:
            self._eng.finish()
        finally:
            self._drain(out)

    def name(self) -> str:
        return "erx"

    def emits_normalized_scores(self) -> bool:
        return True

    def config(self) -> ErxConfig:
        return self._cfg

    def state(self) -> ErxState:
        return self._eng.state(0)

    @property
    def engine(self) -> Engine:
        return self._eng


# ---------------------------------------------------------------- input generator (include/erx_datagen.h)
def gen_spec(config_id: int, stream: int = 0) -> L.GenSpecC:
    s = L.GenSpecC()
    if L.lib().erx_gen_preset(config_id, stream, C.byref(s)):
        raise ConfigError(f"unknown BASELINE config id {config_id}")
    return s


def gen_lines(spec, first: int, n: int, threads: int = 0, want_mask: bool = True):
    """Lines [first, first+n) of one synthetic stream: (fp32 [n][P][B], u8 mask [n][P])."""
    out = np.empty((n, spec.pixels, spec.bands), np.float32)
    mask = np.empty((n, spec.pixels), np.uint8) if want_mask else None
    st = L.lib().erx_gen_lines(C.byref(spec), first, n, _p(out, C.c_float),
                               _p(mask, C.c_uint8) if want_mask else C.POINTER(C.c_uint8)(), threads)
    if st:
        raise ConfigError("bad generator spec")
    return out, mask


def gen_scene_changes(spec):
    """The stream's scene-change lines as the generator drew them (sorted)."""
    out = (C.c_int64 * 4)()
    n = L.lib().erx_gen_scene_changes(C.byref(spec), out)
    if n < 0:
        raise ConfigError("bad generator spec")
    return [int(out[i]) for i in range(n)]


def gen_lines_device(spec, first: int, n: int, out=None, mask=None, want_mask: bool = True, stream: int = 0):
    """The same lines generated on the device (erx_gen_lines_device): torch CUDA tensors
    (fp32 [n][P][B], u8 [n][P] or None).  `out` / `mask` may be preallocated (contiguous)."""
    import torch

    if out is None:
        out = torch.empty((n, spec.pixels, spec.bands), dtype=torch.float32, device="cuda")
    if mask is None and want_mask:
        mask = torch.empty((n, spec.pixels), dtype=torch.uint8, device="cuda")
    st = L.lib().erx_gen_lines_device(C.byref(spec), first, n, out.data_ptr(),
                                      mask.data_ptr() if mask is not None else None, stream or None)
    if st:
        _raise(st, f"gen_lines_device: status {st}")
    return out, mask
