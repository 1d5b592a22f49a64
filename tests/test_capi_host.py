"""CPU-only checks of liberx_b200.so: it loads, exports every symbol the
include/*.h headers declare, and its host-side pieces (config validation,
had::Rng restatement, generate_srp, the input generator) are pinned — the
Rng against the reference's own golden vectors.  No kernel runs here."""
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_golden.json")))


@pytest.fixture(scope="module")
def pkg():
    import subprocess

    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2408_14947_b200", "csrc")], check=True)
    import paper_2408_14947_b200 as p

    p.lib()
    return p


def declared_symbols():
    names = set()
    for h in ("erx_b200.h", "erx_datagen.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(erx_[a-z0-9_]+)\s*\(", src):
            names.add(m.group(1))
    return names


def test_exports_every_declared_symbol(pkg):
    import ctypes

    lib = pkg.lib()
    names = declared_symbols()
    assert len(names) >= 30
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    from paper_2408_14947_b200 import _lib

    assert names == set(_lib.SIGNATURES), names ^ set(_lib.SIGNATURES)
    assert isinstance(lib, ctypes.CDLL)


def test_probe_library_exports_its_header(pkg):
    """Design probes and tcgen05 self-tests live in liberx_probe.so (include/erx_probe.h), not in
    the product library."""
    from paper_2408_14947_b200 import probe

    src = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "erx_probe.h")).read(), flags=re.S)
    names = {m.group(1) for m in re.finditer(r"\b(erx_[a-z0-9_]+)\s*\(", src)}
    assert names == set(probe.SIGNATURES)
    lib = probe.lib()
    assert all(hasattr(lib, n) for n in names)
    assert not any(hasattr(pkg.lib(), n) for n in names)


def test_oracle_generator_is_bitwise_the_product_generator(pkg, oracle):
    """The CPU baseline / reference arm generates its inputs with the oracle library's own copy of
    the seeded generator (no product .so mapped): same bits as erx_gen_lines."""
    for cid, s in ((0, 0), (1, 0), (2, 0), (3, 17), (4, 2)):
        a, ma = oracle.gen_lines(oracle.gen_spec(cid, s), 5, 3, threads=2)
        b, mb = pkg.gen_lines(pkg.gen_spec(cid, s), 5, 3, threads=2)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)) and np.array_equal(ma, mb), (cid, s)
        assert oracle.gen_scene_changes(oracle.gen_spec(cid, s)) == pkg.gen_scene_changes(pkg.gen_spec(cid, s))
    assert pkg.gen_scene_changes(pkg.gen_spec(1, 0)) == [5000]
    assert len(pkg.gen_scene_changes(pkg.gen_spec(4, 3))) == 2


def test_config_validation(pkg):  # erx.hpp:23
    pkg.ErxConfig().validate(108)
    for kw in [dict(alpha=0.0), dict(alpha=1.01), dict(epsilon=0.0), dict(dims=0), dict(dims=109)]:
        with pytest.raises(pkg.ConfigError):
            pkg.ErxConfig(**kw).validate(108)
    pkg.ErxConfig(no_srp=True, dims=0).validate(108)  # dims ignored with no_srp (d = b)
    assert pkg.ConfigError("x").exit_code() == GOLD["exit_codes"]["config"]
    assert pkg.DataError("x").exit_code() == GOLD["exit_codes"]["data"]
    assert pkg.FactorizationError(3, "x").exit_code() == GOLD["exit_codes"]["numeric"]
    assert pkg.FactorizationError.kind == GOLD["error_kinds"]["numeric"]


@pytest.mark.parametrize("seed", [0, 1, 42, 0xDEADBEEF])
def test_product_rng_matches_reference_golden(pkg, seed):
    import ctypes as C

    lib = pkg.lib()
    u = np.zeros(16, np.uint64)
    f = np.zeros(17)
    P64 = C.POINTER(C.c_uint64)
    PD = C.POINTER(C.c_double)
    lib.erx_rng_probe(seed, 0, 16, u.ctypes.data_as(P64), f.ctypes.data_as(PD))
    assert [str(int(x)) for x in u] == GOLD[f"next_u64_seed{seed}"]
    lib.erx_rng_probe(seed, 1, 16, u.ctypes.data_as(P64), f.ctypes.data_as(PD))
    assert f[:16].tolist() == GOLD[f"uniform_seed{seed}"]
    lib.erx_rng_probe(seed, 2, 16, u.ctypes.data_as(P64), f.ctypes.data_as(PD))
    assert f[:16].tolist() == GOLD[f"uniform_f32_seed{seed}"]
    lib.erx_rng_probe(seed, 3, 17, u.ctypes.data_as(P64), f.ctypes.data_as(PD))
    np.testing.assert_allclose(f, GOLD[f"normal_seed{seed}"], rtol=1e-15, atol=1e-15)
    assert [str(lib.erx_mix_seed(s, n)) for s in (0, 1, 42, 0xDEADBEEF)
            for n in (0, 1, 2, 99, 5000, 0xFFFFFFFFFFFFFFFF)] == GOLD["mix_seed"]


def test_generate_srp_matches_oracle(pkg, oracle):
    for b, d, seed in [(108, 5, 0), (224, 5, 3), (10, 5, 9), (100, 5, 123), (1, 1, 5)]:
        np.testing.assert_array_equal(pkg.generate_srp(b, d, seed), oracle.generate_srp(b, d, seed))


def test_generator_deterministic_and_parallel(pkg):
    spec = pkg.gen_spec(0)
    a, ma = pkg.gen_lines(spec, 0, 24, threads=1)
    b, mb = pkg.gen_lines(spec, 0, 24, threads=8)
    c, mc = pkg.gen_lines(spec, 10, 14, threads=3)
    assert np.array_equal(a, b) and np.array_equal(ma, mb)
    assert np.array_equal(a[10:], c) and np.array_equal(ma[10:], mc)
    assert a.dtype == np.float32 and a.shape == (24, 384, 108)
    assert np.isfinite(a).all() and 0.0 < a.mean() < 0.7


@pytest.mark.parametrize("cid", [0, 1, 2, 3, 4])
def test_generator_presets_shapes_and_anomaly_density(pkg, cid):
    spec = pkg.gen_spec(cid, 1)
    dims = {0: (2000, 384, 108), 1: (10000, 640, 224), 2: (20000, 1024, 10), 3: (5000, 640, 108),
            4: (3000, 1280, 448)}[cid]
    assert (spec.lines, spec.pixels, spec.bands) == dims
    n = 40 if cid != 4 else 12
    x, m = pkg.gen_lines(spec, 0, n)
    assert x.shape == (n, dims[1], dims[2]) and np.isfinite(x).all()
    frac = {0: 0.003, 1: 0.002, 2: 0.005, 3: 0.003, 4: 0.002}[cid]
    big = pkg.gen_lines(spec, 0, min(spec.lines, 400), want_mask=True)[1] if cid != 4 else m
    assert big.mean() < 10 * frac + 0.01
