"""Oracle equivalence against an independent dense numpy restatement.

SPEC.md:310 ([DERIVED] random 200-line stream: every delta matches a dense
oracle computing sqrt((z-mu)^T (K+eps I)^{-1} (z-mu)) with explicitly
maintained EMA statistics, within 1e-8) and acceptance criterion 1
(50 random small streams, p <= 20, b <= 8, 300 lines, 1e-7).
"""
import numpy as np
import pytest


def dense_erx(lines, alpha, eps, w=None, incremental=False):
    mu = cov = None
    n_seen = 0
    raws = []
    for x in lines:
        z = x.astype(np.float64) if w is None else x.astype(np.float64) @ w
        p = z.shape[0]
        mh = z.mean(0)
        kh = (z - mh).T @ (z - mh) / (p - 1)
        first = mu is None
        if first:
            mu, cov, n_seen = mh.copy(), kh.copy(), p
        e = eps
        while True:
            a = cov + e * np.eye(z.shape[1])
            if np.all(np.linalg.eigvalsh(a) > 0):
                break
            e *= 10
        v = z - mu
        raws.append(np.sqrt(np.einsum("ij,ij->i", v, np.linalg.solve(a, v.T).T)))
        if not first:
            if incremental:
                n2 = n_seen + p
                d = mh - mu
                cov = (cov * (n_seen - 1) + kh * (p - 1) + np.outer(d, d) * n_seen * p / n2) / (n2 - 1)
                mu = mu + d * p / n2
                n_seen = n2
            else:
                mu = (1 - alpha) * mu + alpha * mh
                cov = (1 - alpha) * cov + alpha * kh
    return np.array(raws)


def test_dense_200_lines_1e8(oracle):
    rng = np.random.default_rng(20)
    lines = rng.uniform(size=(200, 16, 5)).astype(np.float32)
    raw, _, _ = oracle.run_stream(oracle.OracleConfig(no_srp=True, alpha=0.1), lines)
    ref = dense_erx(lines, 0.1, 1e-5)
    assert np.max(np.abs(raw - ref) / np.maximum(ref, 1e-300)) <= 1e-8


@pytest.mark.parametrize("incremental", [False, True])
def test_acceptance_1_fifty_streams(oracle, incremental):
    rng = np.random.default_rng(21 + incremental)
    worst = 0.0
    for s in range(50):
        p = int(rng.integers(9, 21))
        b = int(rng.integers(2, 9))
        alpha = float(rng.choice([1.0, 0.5, 0.1, 0.01]))
        lines = (rng.uniform(size=(300, p, b)) + np.linspace(0, 1, 300)[:, None, None]).astype(np.float32)
        use_srp = bool(s % 2)
        cfg = oracle.OracleConfig(no_srp=not use_srp, dims=max(1, b // 2), alpha=alpha, seed=s,
                                  use_incremental=incremental)
        raw, _, det = oracle.run_stream(cfg, lines)
        w = det.state()["weights"] if use_srp else None
        ref = dense_erx(lines, alpha, 1e-5, w=w, incremental=incremental)
        worst = max(worst, float(np.max(np.abs(raw - ref) / np.maximum(ref, 1e-12))))
    assert worst <= 1e-7
