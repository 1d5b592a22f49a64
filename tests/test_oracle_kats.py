"""SPEC.md known-answer tests and properties, run against the CPU oracle.

Every test names the SPEC.md line(s) whose [TRIVIAL]/[DERIVED]/[PAPER]
example or invariant it encodes.  These pin the oracle before it is trusted
as the checker for the CUDA path (tests/test_gpu_parity.py).
"""
import math

import numpy as np
import pytest


def spd(rng, n, cond=10.0):
    q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    ev = np.exp(rng.uniform(0, math.log(cond), n))
    return (q * ev) @ q.T


# ---------------------------------------------------------------- linalg
def test_cholesky_kats(oracle):
    l, piv = oracle.cholesky_lower(np.eye(3))
    assert piv == -1 and np.array_equal(l, np.eye(3))
    l, piv = oracle.cholesky_lower(np.array([[4.0, 2.0], [2.0, 3.0]]))
    assert piv == -1
    np.testing.assert_allclose(l, [[2, 0], [1, math.sqrt(2)]], rtol=0, atol=1e-15)
    rng = np.random.default_rng(0)
    a = spd(rng, 5)
    l, piv = oracle.cholesky_lower(a)
    assert piv == -1 and np.allclose(l @ l.T, a, rtol=1e-10, atol=1e-12)


def test_cholesky_reads_lower_triangle_and_reports_pivot(oracle):  # linalg.hpp:12-15
    a = np.array([[4.0, 999.0], [2.0, 3.0]])
    l, piv = oracle.cholesky_lower(a)
    np.testing.assert_allclose(l, [[2, 0], [1, math.sqrt(2)]], atol=1e-15)
    bad = np.array([[1.0, 0, 0], [0, 1.0, 0], [0, 2.0, 1.0]])  # not PD: fails at pivot 2
    _, piv = oracle.cholesky_lower(bad)
    assert piv == 2
    _, piv = oracle.cholesky_lower(np.array([[float("nan")]]))
    assert piv == 0


def test_forward_substitute_kats(oracle):
    x, st = oracle.forward_substitute(np.eye(3), [1, 2, 3])
    assert st == -1 and np.array_equal(x, [1, 2, 3])
    x, st = oracle.forward_substitute(np.array([[2.0, 0], [1, math.sqrt(2)]]), [2, 1])
    np.testing.assert_allclose(x, [1, 0], atol=1e-15)
    rng = np.random.default_rng(1)
    for _ in range(50):
        n = int(rng.integers(1, 17))
        l = np.tril(rng.normal(size=(n, n))) + np.eye(n) * 3
        v = rng.normal(size=n)
        m, st = oracle.forward_substitute(l, v)
        assert st == -1 and np.linalg.norm(l @ m - v) <= 1e-10 * max(1, np.linalg.norm(v))
    _, st = oracle.forward_substitute(np.array([[1.0, 0], [1, 0.0]]), [1, 1])
    assert st == 1  # SingularSolveError on the zero diagonal (linalg.hpp:17)


def test_linalg_randomized_1000(oracle):  # SPEC.md:175-177 (1,000 instances, n <= 16)
    rng = np.random.default_rng(2)
    for _ in range(1000):
        n = int(rng.integers(1, 17))
        a = spd(rng, n, cond=100.0)
        l, piv = oracle.cholesky_lower(a)
        assert piv == -1
        assert np.allclose(l @ l.T, a, rtol=1e-10, atol=1e-12 * np.abs(a).max())
        v = rng.normal(size=n)
        m, _ = oracle.forward_substitute(l, v)
        q = v @ np.linalg.solve(a, v)
        assert abs(m @ m - q) <= 1e-8 * abs(q)


def test_welford_kats(oracle):
    rng = np.random.default_rng(3)
    x = rng.normal(size=(7, 4))
    mean, cov, n, st = oracle.welford_batch_update(np.zeros(4), np.zeros((4, 4)), 0, x)
    assert st == 0 and n == 7
    np.testing.assert_allclose(mean, x.mean(0), rtol=1e-12)
    np.testing.assert_allclose(cov, np.cov(x.T), rtol=1e-10, atol=1e-14)
    c = np.tile([1.5, -2.0, 3.0], (5, 1))
    m2, c2, n2, _ = oracle.welford_batch_update(np.zeros(3), np.zeros((3, 3)), 0, c)
    m2, c2, n2, _ = oracle.welford_batch_update(m2, c2, n2, c)
    assert n2 == 10 and np.abs(c2).max() == 0.0
    batches = [rng.normal(size=(int(rng.integers(1, 9)), 5)) for _ in range(10)]
    mean, cov, n = np.zeros(5), np.zeros((5, 5)), 0
    for b in batches:
        mean, cov, n, _ = oracle.welford_batch_update(mean, cov, n, b)
    allx = np.concatenate(batches)
    np.testing.assert_allclose(mean, allx.mean(0), rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(cov, np.cov(allx.T), rtol=1e-8, atol=1e-12)


# ---------------------------------------------------------------- projection
def test_srp_law_b100_d5(oracle):  # SPEC.md:216, acceptance criterion 3
    counts = []
    for seed in range(200):
        w = oracle.generate_srp(100, 5, seed)
        v = math.sqrt(10.0) / math.sqrt(5.0)
        assert set(np.unique(np.abs(w))) <= {0.0, v}
        counts.append(int((w != 0).sum()))
    sigma = math.sqrt(500 * 0.1 * 0.9)
    assert abs(counts[0] - 50) <= 3 * sigma
    assert abs(np.mean(counts) - 50) <= 3 * sigma / math.sqrt(200)
    zero_frac = 1 - np.mean(counts) / 500
    assert abs(zero_frac - 0.9) <= 3 * math.sqrt(0.09 / (500 * 200))


def test_srp_trivial(oracle):
    vals = {float(oracle.generate_srp(1, 1, s)[0, 0]) for s in range(64)}
    assert vals == {1.0, -1.0}
    assert np.array_equal(oracle.generate_srp(108, 5, 7), oracle.generate_srp(108, 5, 7))
    assert not np.array_equal(oracle.generate_srp(108, 5, 7), oracle.generate_srp(108, 5, 8))


def test_project_line(oracle):
    rng = np.random.default_rng(4)
    x = rng.uniform(size=(6, 9)).astype(np.float32)
    z, st = oracle.project_line(x, np.zeros((9, 3)))
    assert st == 0 and np.abs(z).max() == 0.0
    w = np.zeros((9, 3))
    w[4, 1] = 2.5
    z, _ = oracle.project_line(x, w)
    np.testing.assert_array_equal(z[:, 1], 2.5 * x[:, 4].astype(np.float64))
    w = oracle.generate_srp(9, 3, 1)
    z, _ = oracle.project_line(x, w)
    naive = np.array([[sum(float(x[i, k]) * w[k, j] for k in range(9)) for j in range(3)] for i in range(6)])
    np.testing.assert_allclose(z, naive, rtol=1e-12, atol=1e-12)
    y = rng.uniform(size=(6, 9)).astype(np.float32)
    za, _ = oracle.project_line(x, w)
    zb, _ = oracle.project_line(y, w)
    zs, _ = oracle.project_line((x.astype(np.float64) + y).astype(np.float32), w)
    np.testing.assert_allclose(zs, za + zb, rtol=1e-6, atol=1e-6)
    _, st = oracle.project_line(x, np.zeros((8, 3)))
    assert st == 2  # ConfigError on band mismatch (projection.hpp:31-32)


# ---------------------------------------------------------------- erx free functions
def test_line_stats_kats(oracle):
    mu, cov, st = oracle.line_stats(np.array([[0.0, 0.0], [2.0, 2.0]]))
    assert st == 0
    np.testing.assert_array_equal(mu, [1, 1])
    np.testing.assert_array_equal(cov, [[2, 2], [2, 2]])
    mu, cov, _ = oracle.line_stats(np.tile([3.0, 1.0, 2.0], (5, 1)))
    assert np.abs(cov).max() == 0.0
    rng = np.random.default_rng(5)
    z = rng.normal(size=(50, 5))
    mu, cov, _ = oracle.line_stats(z)
    np.testing.assert_allclose(mu, z.mean(0), rtol=1e-10)
    np.testing.assert_allclose(cov, np.cov(z.T), rtol=1e-10, atol=1e-14)
    _, _, st = oracle.line_stats(np.ones((1, 3)))
    assert st == 3  # DataError for p < 2 (erx.hpp:39)


def test_normalize_and_threshold(oracle):  # detector.hpp:29-32
    assert np.array_equal(oracle.normalize_scores(np.full(7, 3.25)), np.zeros(7))
    rng = np.random.default_rng(6)
    n = oracle.normalize_scores(rng.gamma(2.0, size=333))
    assert abs(n.mean()) < 1e-9 and abs(n.std() - 1.0) < 1e-9
    s = np.array([-1.0, 0.0, 2.0])
    assert oracle.apply_threshold(s, -np.inf).tolist() == [1, 1, 1]
    assert oracle.apply_threshold(s, np.inf).tolist() == [0, 0, 0]
    assert oracle.apply_threshold(s, 1.0).tolist() == [0, 0, 1]
    taus = np.linspace(-2, 3, 11)
    counts = [oracle.apply_threshold(s, t).sum() for t in taus]
    assert all(a >= b for a, b in zip(counts, counts[1:]))  # monotone


# ---------------------------------------------------------------- detector
def test_detector_init_and_ema(oracle):
    cfg = oracle.OracleConfig(no_srp=True, alpha=0.1)
    det = oracle.OracleErx(cfg, 1)
    raw, norm, wu = det.process(0, np.zeros((4, 1), np.float32))
    st = det.state()
    assert st["initialized"] and st["mu"][0] == 0.0 and st["cov"][0, 0] == 0.0 and wu
    assert np.array_equal(norm, np.zeros(4))
    det.process(1, np.full((4, 1), 10.0, np.float32))
    assert det.state()["mu"][0] == pytest.approx(1.0, abs=1e-15)
    # alpha = 1: state = current line only.
    det1 = oracle.OracleErx(oracle.OracleConfig(no_srp=True, alpha=1.0), 2)
    rng = np.random.default_rng(7)
    det1.process(0, rng.normal(size=(6, 2)).astype(np.float32))
    x = rng.normal(size=(6, 2)).astype(np.float32)
    det1.process(1, x)
    mu, cov, _ = oracle.line_stats(x.astype(np.float64))
    np.testing.assert_allclose(det1.state()["mu"], mu, rtol=1e-15)
    np.testing.assert_allclose(det1.state()["cov"], cov, rtol=1e-14)
    # geometric convergence to a constant mu_hat
    det2 = oracle.OracleErx(oracle.OracleConfig(no_srp=True, alpha=0.1), 1)
    det2.process(0, np.zeros((3, 1), np.float32))
    for n in range(1, 30):
        det2.process(n, np.full((3, 1), 5.0, np.float32))
        assert abs(det2.state()["mu"][0] - 5.0) == pytest.approx(0.9 ** n * 5.0, rel=1e-12)


def test_detector_euclidean_case(oracle):  # SPEC.md:308 (K + eps I = I, z - mu = (3,4) -> 5)
    t = math.sqrt(1.5 * (1.0 - 1e-5))
    line0 = np.array([[t, 0], [-t, 0], [0, t], [0, -t]], np.float32)
    det = oracle.OracleErx(oracle.OracleConfig(no_srp=True, alpha=0.1), 2)
    det.process(0, line0)
    raw, _, _ = det.process(1, np.array([[3, 4], [0, 0], [1, 0]], np.float32))
    assert raw[0] == pytest.approx(5.0, rel=1e-6) and raw[1] == pytest.approx(0.0, abs=1e-6)


def test_detector_config_errors(oracle):  # erx.hpp:23
    for kw in [dict(alpha=0.0), dict(alpha=1.5), dict(epsilon=0.0), dict(dims=0), dict(dims=200)]:
        with pytest.raises(oracle.OracleError) as e:
            oracle.OracleErx(oracle.OracleConfig(**kw), 108)
        assert e.value.code == 2
    det = oracle.OracleErx(oracle.OracleConfig(), 10)
    with pytest.raises(oracle.OracleError) as e:
        det.process(0, np.zeros((5, 9), np.float32))
    assert e.value.code == 2
    with pytest.raises(oracle.OracleError) as e:
        det.process(0, np.zeros((1, 10), np.float32))
    assert e.value.code == 3


def test_detector_factorization_error(oracle):  # SPEC.md:306, errors.hpp:51-56
    det = oracle.OracleErx(oracle.OracleConfig(no_srp=True), 3)
    x = np.random.default_rng(0).normal(size=(8, 3)).astype(np.float32)
    x[0, 1] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        det.process(0, x)
    assert e.value.code == 5 and e.value.pivot >= 0


def test_warmup_flag(oracle):
    det = oracle.OracleErx(oracle.OracleConfig(buffer_len=3), 6)
    rng = np.random.default_rng(9)
    flags = [det.process(t, rng.uniform(size=(10, 6)).astype(np.float32))[2] for t in range(5)]
    assert flags == [True, True, True, False, False]


def test_score_then_update(oracle):
    rng = np.random.default_rng(10)
    det = oracle.OracleErx(oracle.OracleConfig(no_srp=True), 4)
    for t in range(20):
        raw, _, _ = det.process(t, rng.normal(0, 0.1, (30, 4)).astype(np.float32))
    bg = raw.mean()
    raw, _, _ = det.process(20, (rng.normal(0, 0.1, (30, 4)) + 5.0).astype(np.float32))
    assert raw.min() > 10 * bg


def test_adaptation_property(oracle):
    rng = np.random.default_rng(11)
    alpha = 0.1
    det = oracle.OracleErx(oracle.OracleConfig(no_srp=True, alpha=alpha), 3)
    pre = []
    for t in range(100):
        raw, _, _ = det.process(t, rng.normal(0, 0.1, (40, 3)).astype(np.float32))
        pre.extend(raw)
    p95 = np.percentile(pre[-40 * 50:], 95)
    n_lines = math.ceil(math.log(0.01) / math.log(1 - alpha))
    for k in range(n_lines):
        raw, _, _ = det.process(100 + k, (rng.normal(0, 0.1, (40, 3)) + 1.0).astype(np.float32))
    assert np.median(raw) < p95


# ---------------------------------------------------------------- metrics
def test_roc_auc_kats(oracle):
    s = np.array([0.9, 0.8, 0.1, 0.2])
    assert oracle.roc_auc(s, [1, 1, 0, 0]) == 1.0
    assert oracle.roc_auc(s, [0, 0, 1, 1]) == 0.0
    rng = np.random.default_rng(12)
    for _ in range(100):
        n = 200
        sc = np.round(rng.normal(size=n), 1)  # ties on purpose
        y = (rng.uniform(size=n) < 0.3).astype(np.uint8)
        if y.min() == y.max():
            continue
        pos, neg = sc[y == 1], sc[y == 0]
        mw = ((pos[:, None] > neg[None, :]).sum() + 0.5 * (pos[:, None] == neg[None, :]).sum()) / (pos.size * neg.size)
        assert abs(oracle.roc_auc(sc, y) - mw) <= 1e-10
        assert abs(oracle.roc_auc(sc, y) + oracle.roc_auc(-sc, y) - 1.0) <= 1e-12
    with pytest.raises(oracle.OracleError):
        oracle.roc_auc([1.0, 2.0], [1, 1])
