"""ctypes bindings for the CPU fp64 oracle (oracle/erx_oracle.h).

TEST INFRASTRUCTURE ONLY: imported by tests/, by __graft_entry__.smoke() as
the checker, and by bench.py's cpu_baseline / --impl reference leg.  The
product package (paper_2408_14947_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liberx_oracle.so")
_lib = None


class OrcConfig(C.Structure):
    _fields_ = [
        ("dims", C.c_int32),
        ("alpha", C.c_double),
        ("buffer_len", C.c_uint32),
        ("epsilon", C.c_double),
        ("seed", C.c_uint64),
        ("no_srp", C.c_int32),
        ("use_incremental", C.c_int32),
    ]


class GenSpec(C.Structure):
    """erx_gen_spec (include/erx_datagen.h): the seeded BASELINE.json generator's parameters."""
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


def build() -> str:
    """Compile the oracle library (g++ only; seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE, "all"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        dp = C.POINTER(C.c_double)
        fp = C.POINTER(C.c_float)
        u8p = C.POINTER(C.c_uint8)
        L.orc_rng_new.restype = C.c_void_p
        L.orc_rng_new.argtypes = [C.c_uint64]
        L.orc_rng_free.argtypes = [C.c_void_p]
        for n, rt in [("orc_rng_next_u64", C.c_uint64), ("orc_rng_uniform", C.c_double),
                      ("orc_rng_uniform_f32", C.c_float), ("orc_rng_normal", C.c_double)]:
            getattr(L, n).restype = rt
            getattr(L, n).argtypes = [C.c_void_p]
        L.orc_rng_below.restype = C.c_uint64
        L.orc_rng_below.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_rng_sample_indices.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32),
                                             C.POINTER(C.c_uint32)]
        L.orc_mix_seed.restype = C.c_uint64
        L.orc_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_cholesky_lower.restype = C.c_int
        L.orc_cholesky_lower.argtypes = [dp, C.c_int, dp]
        L.orc_forward_substitute.restype = C.c_int
        L.orc_forward_substitute.argtypes = [dp, C.c_int, dp]
        L.orc_welford_batch_update.restype = C.c_int
        L.orc_welford_batch_update.argtypes = [dp, dp, C.POINTER(C.c_int64), dp, C.c_int, C.c_int]
        L.orc_generate_srp.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, dp]
        L.orc_project_line.restype = C.c_int
        L.orc_project_line.argtypes = [fp, C.c_uint32, C.c_uint32, dp, C.c_uint32, C.c_uint32, C.c_int, dp]
        L.orc_line_stats.restype = C.c_int
        L.orc_line_stats.argtypes = [dp, C.c_int, C.c_int, dp, dp]
        L.orc_normalize_scores.argtypes = [dp, C.c_int, dp]
        L.orc_apply_threshold.argtypes = [dp, C.c_int, C.c_double, u8p]
        L.orc_erx_new.restype = C.c_void_p
        L.orc_erx_new.argtypes = [C.POINTER(OrcConfig), C.c_uint32, C.POINTER(C.c_int), C.c_char_p, C.c_size_t]
        L.orc_erx_free.argtypes = [C.c_void_p]
        L.orc_erx_dims.restype = C.c_int
        L.orc_erx_dims.argtypes = [C.c_void_p]
        L.orc_erx_process.restype = C.c_int
        L.orc_erx_process.argtypes = [C.c_void_p, C.c_int64, C.c_uint32, C.c_uint32, fp, dp, dp, u8p,
                                      C.POINTER(C.c_int), C.c_char_p, C.c_size_t]
        L.orc_erx_state.restype = C.c_int
        L.orc_erx_state.argtypes = [C.c_void_p, dp, dp, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int), dp]
        L.orc_erx_run_streams.restype = C.c_int
        L.orc_erx_run_streams.argtypes = [C.POINTER(OrcConfig), C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                          fp, dp, dp, C.c_int]
        L.orc_erx_set_state.restype = C.c_int
        L.orc_erx_set_state.argtypes = [C.c_void_p, dp, dp, C.c_int64, C.c_int64]
        L.orc_gen_preset.restype = C.c_int
        L.orc_gen_preset.argtypes = [C.c_int, C.c_uint32, C.c_void_p]
        L.orc_gen_lines.restype = C.c_int
        L.orc_gen_lines.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, fp, u8p, C.c_int]
        L.orc_gen_scene_changes.restype = C.c_int
        L.orc_gen_scene_changes.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
        L.orc_roc_auc.restype = C.c_double
        L.orc_roc_auc.argtypes = [dp, u8p, C.c_size_t, C.POINTER(C.c_int)]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str, pivot: int = -1):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.pivot = pivot


class Rng:
    def __init__(self, seed: int):
        self._h = lib().orc_rng_new(seed)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_rng_free(self._h)

    def next_u64(self):
        return lib().orc_rng_next_u64(self._h)

    def uniform(self):
        return lib().orc_rng_uniform(self._h)

    def uniform_f32(self):
        return lib().orc_rng_uniform_f32(self._h)

    def below(self, b):
        return lib().orc_rng_below(self._h, b)

    def normal(self):
        return lib().orc_rng_normal(self._h)

    def sample_indices(self, n, k):
        out = np.zeros(max(n, 1), np.uint32)
        kk = C.c_uint32(0)
        lib().orc_rng_sample_indices(self._h, n, k, _p(out, C.c_uint32), C.byref(kk))
        return out[: kk.value].tolist()


def mix_seed(seed: int, n: int) -> int:
    return lib().orc_mix_seed(seed, n)


def cholesky_lower(a: np.ndarray):
    a = np.ascontiguousarray(a, np.float64)
    n = a.shape[0]
    l = np.zeros_like(a)
    piv = lib().orc_cholesky_lower(_p(a, C.c_double), n, _p(l, C.c_double))
    return l, piv


def forward_substitute(l: np.ndarray, v: np.ndarray):
    l = np.ascontiguousarray(l, np.float64)
    x = np.array(v, np.float64)
    st = lib().orc_forward_substitute(_p(l, C.c_double), l.shape[0], _p(x, C.c_double))
    return x, st


def welford_batch_update(mean, cov, n_seen, batch):
    mean = np.array(mean, np.float64)
    cov = np.array(cov, np.float64)
    batch = np.ascontiguousarray(batch, np.float64)
    n = C.c_int64(n_seen)
    st = lib().orc_welford_batch_update(_p(mean, C.c_double), _p(cov, C.c_double), C.byref(n),
                                        _p(batch, C.c_double), batch.shape[0], batch.shape[1])
    return mean, cov, n.value, st


def generate_srp(bands: int, dims: int, seed: int) -> np.ndarray:
    w = np.zeros((bands, dims), np.float64)
    lib().orc_generate_srp(bands, dims, seed, _p(w, C.c_double))
    return w


def project_line(x: np.ndarray, w: np.ndarray, identity=False):
    x = np.ascontiguousarray(x, np.float32)
    w = np.ascontiguousarray(w, np.float64)
    p, b = x.shape
    d = b if identity else w.shape[1]
    z = np.zeros((p, d), np.float64)
    st = lib().orc_project_line(_p(x, C.c_float), p, b, _p(w, C.c_double), w.shape[0], d, int(identity),
                                _p(z, C.c_double))
    return z, st


def line_stats(z: np.ndarray):
    z = np.ascontiguousarray(z, np.float64)
    p, d = z.shape
    mu = np.zeros(d)
    cov = np.zeros((d, d))
    st = lib().orc_line_stats(_p(z, C.c_double), p, d, _p(mu, C.c_double), _p(cov, C.c_double))
    return mu, cov, st


def normalize_scores(raw):
    raw = np.ascontiguousarray(raw, np.float64)
    out = np.zeros_like(raw)
    lib().orc_normalize_scores(_p(raw, C.c_double), raw.size, _p(out, C.c_double))
    return out


def apply_threshold(norm, tau):
    norm = np.ascontiguousarray(norm, np.float64)
    out = np.zeros(norm.size, np.uint8)
    lib().orc_apply_threshold(_p(norm, C.c_double), norm.size, tau, _p(out, C.c_uint8))
    return out


def roc_auc(scores, labels):
    s = np.ascontiguousarray(scores, np.float64).ravel()
    y = np.ascontiguousarray(labels, np.uint8).ravel()
    st = C.c_int(0)
    a = lib().orc_roc_auc(_p(s, C.c_double), _p(y, C.c_uint8), s.size, C.byref(st))
    if st.value:
        raise OracleError(st.value, "AUC undefined: need both classes")
    return a


@dataclass
class OracleConfig:
    dims: int = 5
    alpha: float = 0.1
    buffer_len: int = 99
    epsilon: float = 1e-5
    seed: int = 0
    no_srp: bool = False
    use_incremental: bool = False

    def c(self) -> OrcConfig:
        return OrcConfig(self.dims, self.alpha, self.buffer_len, self.epsilon, self.seed, int(self.no_srp),
                         int(self.use_incremental))


class OracleErx:
    """fp64 CPU restatement of had::ErxDetector (erx.hpp:56-71)."""

    def __init__(self, cfg: OracleConfig, bands: int):
        st = C.c_int(0)
        msg = C.create_string_buffer(256)
        self._cfg = cfg.c()
        self._h = lib().orc_erx_new(C.byref(self._cfg), bands, C.byref(st), msg, 256)
        if not self._h:
            raise OracleError(st.value, msg.value.decode())
        self.bands = bands
        self.dims = lib().orc_erx_dims(self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_erx_free(self._h)

    def process(self, index: int, line: np.ndarray):
        x = np.ascontiguousarray(line, np.float32)
        p, b = x.shape
        raw = np.zeros(p)
        norm = np.zeros(p)
        wu = np.zeros(1, np.uint8)
        piv = C.c_int(-1)
        msg = C.create_string_buffer(256)
        st = lib().orc_erx_process(self._h, index, p, b, _p(x, C.c_float), _p(raw, C.c_double),
                                   _p(norm, C.c_double), _p(wu, C.c_uint8), C.byref(piv), msg, 256)
        if st:
            raise OracleError(st, msg.value.decode(), piv.value)
        return raw, norm, bool(wu[0])

    def set_state(self, mu, cov, lines_seen: int, welford_n: int = 0):
        mu = np.ascontiguousarray(mu, np.float64)
        cov = np.ascontiguousarray(cov, np.float64)
        lib().orc_erx_set_state(self._h, _p(mu, C.c_double), _p(cov, C.c_double), lines_seen, welford_n)

    def state(self):
        d = self.dims
        mu = np.zeros(d)
        cov = np.zeros((d, d))
        ls = C.c_int64(0)
        wn = C.c_int64(0)
        ini = C.c_int(0)
        w = np.zeros((self.bands, d)) if not self._cfg.no_srp else np.zeros((1, 1))
        lib().orc_erx_state(self._h, _p(mu, C.c_double), _p(cov, C.c_double), C.byref(ls), C.byref(wn),
                            C.byref(ini), _p(w, C.c_double))
        return dict(mu=mu, cov=cov, lines_seen=ls.value, welford_n=wn.value, initialized=bool(ini.value),
                    weights=None if self._cfg.no_srp else w)


def gen_spec(config_id: int, stream: int = 0) -> GenSpec:
    """BASELINE.json configs[config_id] generator spec for one stream (erx_gen_preset)."""
    s = GenSpec()
    if lib().orc_gen_preset(config_id, stream, C.byref(s)):
        raise OracleError(2, f"unknown BASELINE config id {config_id}")
    return s


def gen_lines(spec: GenSpec, first: int, n: int, threads: int = 0, want_mask: bool = True):
    """Lines [first, first+n) of one synthetic stream: (fp32 [n][P][B], u8 mask [n][P] or None)."""
    out = np.empty((n, spec.pixels, spec.bands), np.float32)
    mask = np.empty((n, spec.pixels), np.uint8) if want_mask else None
    st = lib().orc_gen_lines(C.byref(spec), first, n, _p(out, C.c_float),
                             _p(mask, C.c_uint8) if want_mask else C.POINTER(C.c_uint8)(), threads)
    if st:
        raise OracleError(st, "bad generator spec")
    return out, mask


def gen_scene_changes(spec: GenSpec):
    """The stream's scene-change lines as the generator drew them (sorted)."""
    out = (C.c_int64 * 4)()
    n = lib().orc_gen_scene_changes(C.byref(spec), out)
    if n < 0:
        raise OracleError(2, "bad generator spec")
    return [int(out[i]) for i in range(n)]


def run_stream(cfg: OracleConfig, lines: np.ndarray):
    """lines: [L][P][B] fp32 -> raw, norm [L][P] fp64."""
    det = OracleErx(cfg, lines.shape[2])
    raw = np.zeros(lines.shape[:2])
    norm = np.zeros(lines.shape[:2])
    for t in range(lines.shape[0]):
        raw[t], norm[t], _ = det.process(t, lines[t])
    return raw, norm, det


def run_streams(cfg: OracleConfig, lines: np.ndarray, threads: int = 1, want_scores: bool = True):
    """lines: [S][L][P][B] fp32, one stream per host thread."""
    x = np.ascontiguousarray(lines, np.float32)
    S, L, P, B = x.shape
    c = cfg.c()
    raw = np.zeros((S, L, P)) if want_scores else None
    norm = np.zeros((S, L, P)) if want_scores else None
    nul = C.POINTER(C.c_double)()
    st = lib().orc_erx_run_streams(C.byref(c), B, S, L, P, _p(x, C.c_float),
                                   _p(raw, C.c_double) if want_scores else nul,
                                   _p(norm, C.c_double) if want_scores else nul, threads)
    if st:
        raise OracleError(st, "oracle stream run failed")
    return raw, norm
