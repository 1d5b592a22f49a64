"""Device generator (csrc/k_datagen.cu) against the host
generator (erx_gen_lines, the bench's and the parity tests' input source).

Masks are identical.  Values are identical except where CUDA's fp64
log / sin / cos round differently from glibc in the last place; after the
fp32 rounding of x such a value differs by exactly one fp32 ulp.  The gate:
no value off by more than one ulp and at most 1e-5 of all values off at all.
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


def ulp_diff(a, b):
    ia = a.view(np.int32).astype(np.int64)
    ib = b.view(np.int32).astype(np.int64)
    ia = np.where(ia < 0, -(ia & 0x7FFFFFFF), ia)  # sign-magnitude -> ordered
    ib = np.where(ib < 0, -(ib & 0x7FFFFFFF), ib)
    return np.abs(ia - ib)


# (config, stream, first line, lines): every anomaly kind, scene changes (c1 at line 5000, c4 drawn),
# R + B odd (c2: Box-Muller pairs straddle pixels), chunk boundaries of the kernel launch
CASES = [(0, 0, 0, 40), (0, 0, 1990, 10), (1, 0, 4990, 20), (2, 0, 100, 64), (3, 17, 2500, 33), (4, 2, 0, 6),
         (4, 1, 1400, 4)]


@pytest.mark.parametrize("cid,stream,first,n", CASES)
def test_device_generator_matches_host(torch_cuda, cid, stream, first, n):
    import paper_2408_14947_b200 as pkg

    spec = pkg.gen_spec(cid, stream)
    xh, mh = pkg.gen_lines(spec, first, n)
    xd, md = pkg.gen_lines_device(spec, first, n)
    xd, md = xd.cpu().numpy(), md.cpu().numpy()
    np.testing.assert_array_equal(md, mh)
    d = ulp_diff(xd, xh)
    assert d.max() <= 1, f"max ulp diff {d.max()}"
    assert np.count_nonzero(d) <= max(1, int(1e-5 * d.size)), f"{np.count_nonzero(d)} of {d.size} differ"


def test_device_generator_anomalies_present(torch_cuda):
    """c0 lines 0..299 contain blobs: the mask marks them on both paths."""
    import paper_2408_14947_b200 as pkg

    spec = pkg.gen_spec(0, 0)
    _, md = pkg.gen_lines_device(spec, 0, 300)
    _, mh = pkg.gen_lines(spec, 0, 300)
    assert int(mh.sum()) > 0
    np.testing.assert_array_equal(md.cpu().numpy(), mh)


def test_device_generator_feeds_engine(torch_cuda):
    """A c3 window generated on the device and scored in place equals the host-fed run's scores."""
    import paper_2408_14947_b200 as pkg

    torch = torch_cuda
    spec = pkg.gen_spec(3, 5)
    n, P, B = 64, spec.pixels, spec.bands
    xd, _ = pkg.gen_lines_device(spec, 0, n)
    xh, _ = pkg.gen_lines(spec, 0, n)
    same_input = ulp_diff(xd.cpu().numpy(), xh).max() == 0
    # score the device-generated lines with a device-resident engine, the host lines with another
    outs = []
    for src in (xd, torch.from_numpy(xh).cuda()):
        eng = pkg.Engine(pkg.ErxConfig(alpha=0.1, no_srp=True), B, 1, 32)
        raw = torch.empty((32, P), dtype=torch.float32, device="cuda")
        norm = torch.empty_like(raw)
        res = []
        for w in range(n // 32):
            eng.run_device(src[w * 32:(w + 1) * 32].data_ptr(), 32, P, raw.data_ptr(), norm.data_ptr(), w * 32)
            eng.sync()
            res.append(raw.cpu().numpy().copy())
        eng.close()
        outs.append(np.concatenate(res))
    if same_input:
        np.testing.assert_array_equal(outs[0], outs[1])
    else:
        np.testing.assert_allclose(outs[0], outs[1], rtol=1e-5)
