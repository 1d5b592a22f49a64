"""GPU numerics at the edges the reference's contract names, against the fp64 oracle.

* eps escalation: a background K with a negative eigenvalue of
  -5e-5 (installed on both sides with set_state, as a stream could reach it by
  rounding) makes K + 1e-5 I fail and K + 1e-4 I succeed; the engine must pick
  the oracle's eps and score with it, on every kernel path.
* rank-deficient line covariance, P - 1 < D (erx.hpp:38-40: 1/(P-1)), P = 2,
  alpha = 1, radiance-scale (DN) data whose covariance is
  ill-conditioned for fp32 (A_ii / L_ii^2 up to ~2e5).
* the SRP d-sweep of the paper's ablation: d in {1, 3, 10, 20, 30, 50}.
* apply_threshold (erx.hpp:46-47) of the product against the oracle's.

The fp32 factor hands every line it cannot take (failed or ill-conditioned
pivot) to the fp64 rescue (k_fixup.cu); these tests are what pins that path.
"""
import numpy as np
import pytest

from test_gpu_parity import RAW_MAX, RAW_MED, check_gates, ocfg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2408_14947_b200 as p

    p.lib()
    return p


def run_both(pkg, oracle, cfg, x, window=8, state=None, factor=None, want_stats=None):
    """x: [L][P][B] one stream through the engine (host path) and the oracle; state: (mu, K, lines)."""
    L_, P, B = x.shape
    eng = pkg.Engine(cfg, B, window_lines=window)
    if factor is not None:
        eng.set_factor_precision(factor)
    det = oracle.OracleErx(ocfg(oracle, cfg), B)
    if state is not None:
        mu, K, seen = state
        eng.set_state(0, mu, K, lines_seen=seen, welford_n=seen * P if cfg.use_incremental else 0)
        det.set_state(mu, K, seen, seen * P if cfg.use_incremental else 0)
    eng.push(x[None], 0)
    eng.finish()
    _, wu, raw_g, norm_g = eng.pop()
    raw_o = np.zeros((L_, P))
    norm_o = np.zeros((L_, P))
    for t in range(L_):
        raw_o[t], norm_o[t], _ = det.process(t, x[t])
    info = {"stats": eng.stats_tensor(), "factor": eng.factor_precision(), "rescued": eng.rescued_lines()}
    if want_stats is not None:
        assert info["stats"] == want_stats, info
    eng.close()
    return raw_g[0], norm_g[0], raw_o, norm_o, info


def structured_lines(rng, L_, P, B, n_fac=6, scale=1.0, noise=0.01, offset=0.3):
    A = rng.normal(0, 0.05, size=(B, n_fac))
    base = offset + 0.2 * np.sin(np.linspace(0, 3, B))
    x = base + rng.normal(size=(L_, P, n_fac)) @ A.T + rng.normal(0, noise, size=(L_, P, B))
    return (x * scale).astype(np.float32)


# ---------------------------------------------------------------- eps escalation
@pytest.mark.parametrize("B", [8, 40, 108, 224, 300])
def test_forced_eps_escalation(pkg, oracle, B):
    """K with eigenvalues {-5e-5, logspace(-3, -1)}: the oracle escalates 1e-5 -> 1e-4 on the first
    lines (until the EMA of PSD line covariances lifts the negative direction); the engine, whose
    fp32 factor fails there, must do the same in its fp64 rescue and match every score."""
    rng = np.random.default_rng(B)
    P = 2 * B + 64
    x = structured_lines(rng, 12, P, B)
    Q, _ = np.linalg.qr(rng.normal(size=(B, B)))
    lam = np.concatenate([[-5e-5], np.logspace(-3, -1, B - 1)])
    K = (Q * lam) @ Q.T
    K = 0.5 * (K + K.T)
    mu = x[0].mean(0).astype(np.float64)
    # the oracle needs the escalation on line 0 (pin the premise)
    l, piv = oracle.cholesky_lower(K + 1e-5 * np.eye(B))
    assert piv >= 0
    l, piv = oracle.cholesky_lower(K + 1e-4 * np.eye(B))
    assert piv < 0
    cfg = pkg.ErxConfig(no_srp=True, alpha=0.1, buffer_len=0)
    raw_g, norm_g, raw_o, norm_o, info = run_both(pkg, oracle, cfg, x, window=4, state=(mu, K, 50))
    check_gates(oracle, raw_g, norm_g, raw_o, norm_o, label=f"escalation B={B} {info}")
    assert info["rescued"] > 0, info  # the escalation ran in the fp64 rescue


def test_escalation_exhausted_raises_with_pivot(pkg, oracle):
    """A K that no eps <= 1e-1 repairs (eigenvalue -1): FactorizationError with the oracle's pivot."""
    B, P = 16, 64
    rng = np.random.default_rng(3)
    x = structured_lines(rng, 3, P, B)
    K = np.diag(np.concatenate([np.full(5, 1e-2), [-1.0], np.full(B - 6, 1e-2)]))
    mu = x[0].mean(0).astype(np.float64)
    cfg = pkg.ErxConfig(no_srp=True, alpha=0.1, buffer_len=0)
    det = oracle.OracleErx(ocfg(oracle, cfg), B)
    det.set_state(mu, K, 10)
    with pytest.raises(oracle.OracleError) as eo:
        det.process(0, x[0])
    eng = pkg.Engine(cfg, B, window_lines=2)
    eng.set_state(0, mu, K, lines_seen=10)
    with pytest.raises(pkg.FactorizationError) as eg:
        eng.push(x[None], 0)
        eng.finish()
    assert eg.value.pivot == eo.value.pivot == 5


# ---------------------------------------------------------------- degenerate line statistics
@pytest.mark.parametrize("B,P", [(12, 8), (64, 32), (108, 60), (160, 100), (224, 150)])
def test_rank_deficient_lines(pkg, oracle, B, P):
    """P - 1 < D: each line's covariance is rank P - 1; the first lines' backgrounds are
    eps-regularised and far from fp32 territory (every such line takes the fp64 rescue)."""
    rng = np.random.default_rng(B + P)
    x = structured_lines(rng, 24, P, B)
    cfg = pkg.ErxConfig(no_srp=True, alpha=0.1, buffer_len=0)
    raw_g, norm_g, raw_o, norm_o, info = run_both(pkg, oracle, cfg, x, window=8)
    check_gates(oracle, raw_g, norm_g, raw_o, norm_o, label=f"P-1<D B={B} P={P} {info}")


@pytest.mark.parametrize("B", [4, 24, 130])
@pytest.mark.parametrize("incremental", [False, True])
def test_two_pixel_lines(pkg, oracle, B, incremental):
    """P = 2, the smallest line 1/(P-1) allows (erx.hpp:39): rank-1 line covariances."""
    rng = np.random.default_rng(B)
    x = structured_lines(rng, 16, 2, B)
    cfg = pkg.ErxConfig(no_srp=True, alpha=0.5, buffer_len=0, use_incremental=incremental)
    raw_g, norm_g, raw_o, norm_o, info = run_both(pkg, oracle, cfg, x, window=4)
    check_gates(oracle, raw_g, norm_g, raw_o, norm_o, label=f"P=2 B={B} inc={incremental} {info}")


@pytest.mark.parametrize("no_srp", [True, False])
def test_alpha_one(pkg, oracle, no_srp):
    """alpha = 1: the background is the previous line alone."""
    spec = pkg.gen_spec(0)
    x, mask = pkg.gen_lines(spec, 0, 120)
    cfg = pkg.ErxConfig(no_srp=no_srp, alpha=1.0, buffer_len=10)
    raw_g, norm_g, raw_o, norm_o, info = run_both(pkg, oracle, cfg, x, window=16)
    warm = np.zeros(raw_g.shape, bool)
    warm[:10] = True
    check_gates(oracle, raw_g, norm_g, raw_o, norm_o, mask=mask, warm=warm, label=f"alpha=1 {info}")


@pytest.mark.parametrize("B,noise", [(12, 2e-4), (108, 1e-3), (108, 3e-4), (124, 3e-4)])
def test_radiance_scale_ill_conditioned(pkg, oracle, B, noise):
    """Radiance-scale lines (~2000 DN, 3 latent factors, 0.6-3 DN sensor noise): K + eps I has
    A_ii / L_ii^2 of 1e4 - 2e5, where an fp32 Cholesky loses the score (emulated median error
    1e-3 at 7e5) or fails outright; those lines must come out of the fp64 rescue at the gates.
    (Below ~0.5 DN of noise — finer than a 12-bit sensor's own quantisation — the 22-bit
    integer quantisation of the tensor-core statistics becomes the limit.)"""
    rng = np.random.default_rng(int(B + 1e6 * noise))
    P = 640
    A = rng.normal(0, 0.05, size=(B, 3))
    base = 0.3 + 0.2 * np.sin(np.linspace(0, 3, B))
    x = ((base + rng.normal(size=(40, P, 3)) @ A.T + rng.normal(0, noise, size=(40, P, B))) * 3000.0)
    x = x.astype(np.float32)
    cfg = pkg.ErxConfig(no_srp=True, alpha=0.1, buffer_len=0)
    raw_g, norm_g, raw_o, norm_o, info = run_both(pkg, oracle, cfg, x, window=8)
    check_gates(oracle, raw_g, norm_g, raw_o, norm_o, label=f"DN B={B} noise={noise} {info}")
    assert info["rescued"] > 0, info  # the fp64 rescue took the ill-conditioned lines


# ---------------------------------------------------------------- SRP ablation dims
@pytest.mark.parametrize("d", [1, 3, 10, 20, 30, 50])
def test_srp_dims_sweep(pkg, oracle, d):
    """The paper's d ablation {1, 3, 5, 10, 20, 30, 50} on configs[0] lines: d <= 16 takes the
    small path, larger d the FFMA statistics with the fp64 projection."""
    spec = pkg.gen_spec(0)
    x, mask = pkg.gen_lines(spec, 0, 200)
    cfg = pkg.ErxConfig(no_srp=False, dims=d, alpha=0.1, buffer_len=40, seed=d)
    raw_g, norm_g, raw_o, norm_o, info = run_both(pkg, oracle, cfg, x, window=32)
    warm = np.zeros(raw_g.shape, bool)
    warm[:40] = True
    check_gates(oracle, raw_g, norm_g, raw_o, norm_o, mask=mask, warm=warm, label=f"srp d={d} {info}")


def test_apply_threshold_matches_oracle(pkg, oracle):
    """had::erx::apply_threshold (erx.hpp:46-47) on the product's scores."""
    spec = pkg.gen_spec(0)
    x, _ = pkg.gen_lines(spec, 0, 8)
    det = pkg.ErxDetector(pkg.ErxConfig(no_srp=True), spec.bands, window_lines=4)
    out = []
    for t in range(8):
        det.process(pkg.SpectralLine(t, x[t]), out)
    det.finish(out)
    for s in out:
        for tau in (-np.inf, -1.0, 0.0, 1.5, 3.0, np.inf):
            got = pkg.apply_threshold(s.norm, tau)
            assert np.array_equal(np.asarray(got, np.uint8), oracle.apply_threshold(s.norm, tau))
    assert pkg.apply_threshold(np.array([-1.0, 0.0, 2.0]), 1.0).tolist() == [0, 0, 1]
