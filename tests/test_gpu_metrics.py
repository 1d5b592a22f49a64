"""Device parity-gate metrics against the oracle's roc_auc
(oracle/erx_oracle.cpp, restating had::roc_curve, metrics.hpp:25-28) and an
exact integer Mann-Whitney count; top-k against a stable host sort.

AUC: an exact integer ratio on the device, equal to the host Mann-Whitney
count; compared to the oracle's fp64 trapezoid within 1e-12 (1e-9 for the
~1e5-step ROC of the c0 run: the trapezoid rounds once per step).  Top-k: identical mask
(ties at the cutoff to the lower index) and identical cutoff.
"""
import numpy as np
import pytest

from conftest import has_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import torch

    return torch


def mann_whitney(s, y):
    """2 npos nneg AUC as an exact integer (ties count one half)."""
    s = np.asarray(s, np.float64)
    y = np.asarray(y).astype(bool)
    order = np.argsort(s, kind="stable")
    ss, yy = s[order], y[order]
    heads = np.flatnonzero(np.r_[True, ss[1:] != ss[:-1]])
    ends = np.r_[heads[1:], ss.size]
    negc = np.r_[0, np.cumsum(~yy)]
    tot = 0
    for h, e in zip(heads, ends):
        neg = int(negc[e] - negc[h])
        pos = int((e - h) - neg)
        tot += pos * (2 * int(negc[h]) + neg)
    npos = int(y.sum())
    return tot, npos, y.size - npos


def dev(torch, a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


@pytest.mark.parametrize("n,levels,seed", [(1, 0, 0), (7, 3, 1), (2047, 0, 2), (2049, 5, 3), (100_000, 0, 4),
                                           (100_000, 17, 5), (1_300_000, 1000, 6)])
def test_auc_matches_oracle(torch_cuda, oracle, n, levels, seed):
    from paper_2408_14947_b200 import MetricUndefinedError, metrics

    torch = torch_cuda
    rng = np.random.default_rng(seed)
    y = (rng.random(n) < 0.1).astype(np.uint8)
    s = (rng.standard_normal(n) + 1.5 * y).astype(np.float32)
    if levels:  # heavy ties across both classes
        s = np.round(s * levels / 4).astype(np.float32)
    if n > 2 and y.sum() in (0, n):
        y[0], y[1] = 1, 0
    ds, dy = dev(torch, s, torch.float32), dev(torch, y, torch.uint8)
    if 0 < y.sum() < n:
        got = metrics.roc_auc(ds, dy)
        tot, npos, nneg = mann_whitney(s, y)
        assert got == tot / (2.0 * npos * nneg)
        assert abs(got - oracle.roc_auc(s.astype(np.float64), y)) <= 1e-12
    else:
        with pytest.raises(MetricUndefinedError):
            metrics.roc_auc(ds, dy)


def test_auc_select_and_signed_zero(torch_cuda, oracle):
    from paper_2408_14947_b200 import metrics

    torch = torch_cuda
    rng = np.random.default_rng(11)
    n = 300_001
    y = (rng.random(n) < 0.05).astype(np.uint8)
    s = (np.round(rng.standard_normal(n) * 3) + y).astype(np.float32)
    s[rng.random(n) < 0.1] = -0.0  # -0 and +0 are one tie group, as in the oracle's ==
    sel = (rng.random(n) < 0.8).astype(np.uint8)
    got = metrics.roc_auc(dev(torch, s, torch.float32), dev(torch, y, torch.uint8), dev(torch, sel, torch.uint8))
    m = sel.astype(bool)
    ref = oracle.roc_auc(s[m].astype(np.float64), y[m])
    tot, npos, nneg = mann_whitney(s[m], y[m])
    assert got == tot / (2.0 * npos * nneg)
    assert abs(got - ref) <= 1e-12


def test_auc_undefined(torch_cuda):
    from paper_2408_14947_b200 import MetricUndefinedError, metrics

    torch = torch_cuda
    s = dev(torch, np.arange(10, dtype=np.float32), torch.float32)
    with pytest.raises(MetricUndefinedError):
        metrics.roc_auc(s, dev(torch, np.ones(10, np.uint8), torch.uint8))
    with pytest.raises(MetricUndefinedError):
        metrics.roc_auc(s, dev(torch, np.zeros(10, np.uint8), torch.uint8))
    with pytest.raises(MetricUndefinedError):  # nothing selected
        metrics.roc_auc(s, dev(torch, np.r_[np.ones(5), np.zeros(5)].astype(np.uint8), torch.uint8),
                        dev(torch, np.zeros(10, np.uint8), torch.uint8))


@pytest.mark.parametrize("n,k,levels,seed", [(10, 3, 0, 0), (2048, 2048, 0, 1), (100_000, 1000, 0, 2),
                                             (100_000, 1000, 7, 3), (1_000_003, 10_000, 50, 4), (5, 0, 0, 5)])
def test_top_k_matches_stable_sort(torch_cuda, n, k, levels, seed):
    from paper_2408_14947_b200 import metrics

    torch = torch_cuda
    rng = np.random.default_rng(seed)
    s = rng.standard_normal(n).astype(np.float32)
    if levels:
        s = np.round(s * levels).astype(np.float32)
    sel = (rng.random(n) < 0.9).astype(np.uint8)
    k = min(k, int(sel.sum()))  # (2048, 2048): every selected element
    mask, cut = metrics.top_k(dev(torch, s, torch.float32), k, dev(torch, sel, torch.uint8))
    idx = np.flatnonzero(sel)
    order = idx[np.lexsort((idx, -s[idx].astype(np.float64)))]  # descending score, ties by index
    want = np.zeros(n, np.uint8)
    want[order[:k]] = 1
    np.testing.assert_array_equal(mask.cpu().numpy(), want)
    if k:
        assert cut == s[order[k - 1]]


def test_top_k_too_many(torch_cuda):
    from paper_2408_14947_b200 import DataError, metrics

    torch = torch_cuda
    with pytest.raises(DataError):
        metrics.top_k(dev(torch, np.zeros(4, np.float32), torch.float32), 5)


def test_gates_on_device_c0(torch_cuda, oracle):
    """c0 end to end: the pooled non-warmup norm scores of the engine, gated on the device."""
    import paper_2408_14947_b200 as pkg
    from paper_2408_14947_b200 import metrics

    torch = torch_cuda
    spec = pkg.gen_spec(0, 0)
    n = 400
    x, mask = pkg.gen_lines(spec, 0, n)
    cfg = pkg.ErxConfig(alpha=0.1, no_srp=True)
    det = pkg.ErxDetector(cfg, x.shape[2], window_lines=32)
    out = []
    for t in range(n):
        det.process(pkg.SpectralLine(t, x[t]), out)
    det.finish(out)
    norm = np.stack([o.norm for o in out]).astype(np.float32)
    warm = np.array([o.warmup for o in out])
    sel = np.repeat(~warm, norm.shape[1]).astype(np.uint8)
    y = np.asarray(mask, np.uint8).reshape(-1)
    got = metrics.roc_auc(dev(torch, norm.ravel(), torch.float32), dev(torch, y, torch.uint8),
                          dev(torch, sel, torch.uint8))
    ref = oracle.roc_auc(norm[~warm].ravel().astype(np.float64), np.asarray(mask)[~warm].ravel())
    tot, npos, nneg = mann_whitney(norm[~warm].ravel(), np.asarray(mask)[~warm].ravel())
    assert got == tot / (2.0 * npos * nneg)
    assert abs(got - ref) <= 1e-9  # the oracle's fp64 trapezoid rounds once per ROC step (~1e5 steps)
    k = int(np.ceil(0.01 * sel.sum()))
    m, cut = metrics.top_k(dev(torch, norm.ravel(), torch.float32), k, dev(torch, sel, torch.uint8))
    assert int(m.sum().item()) == k
    assert cut == np.sort(norm[~warm].ravel())[::-1][k - 1]
