"""Hardware check of the hand-written tcgen05 path (tc_common.cuh): UMMA
smem descriptors, instruction descriptor, TMEM alloc/ld and mbarrier commit,
plus the 3-way bf16 split with 6 products (liberx_probe.so, include/erx_probe.h)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K", [16, 64, 128])
def test_tcgen05_bf16_gemm(K):
    import torch

    from paper_2408_14947_b200 import probe

    rng = np.random.default_rng(K)
    a = rng.normal(size=(128, K)).astype(np.float32)
    b = rng.normal(size=(128, K)).astype(np.float32)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    for split, tol in ((0, 3e-2), (1, 2e-6)):
        dd = torch.zeros((128, 128), dtype=torch.float32, device="cuda")
        st = probe.lib().erx_tc_selftest(0, None, C.c_void_p(da.data_ptr()), C.c_void_p(db.data_ptr()), K, split,
                                         C.c_void_p(dd.data_ptr()))
        assert st == 0
        d = dd.cpu().numpy().astype(np.float64)
        err = np.abs(d - ref).max() / np.abs(ref).max()
        assert err < tol, (split, err)


def _i8_gemm(a, b, a_mn, ms=512, ks=128, lbo=128, sbo=512):
    import torch

    from paper_2408_14947_b200 import probe

    K, N = a.shape[1], b.shape[0]
    da = torch.from_numpy(a).cuda()
    db = torch.from_numpy(b).cuda()
    dd = torch.zeros((128, N), dtype=torch.int32, device="cuda")
    st = probe.lib().erx_tc_selftest_i8(0, None, C.c_void_p(da.data_ptr()), C.c_void_p(db.data_ptr()), K, N, a_mn,
                                        ms, ks, lbo, sbo, C.c_void_p(dd.data_ptr()))
    assert st == 0
    return dd.cpu().numpy().astype(np.int64)


@pytest.mark.parametrize("K,N", [(32, 112), (128, 112), (64, 128)])
def test_tcgen05_i8_exact(K, N):
    """kind::i8 MMAs accumulate exactly in s32, for K-major and MN-major A operands (the
    MN-major layout is the score kernel's v-plane tile: 16-pixel groups 512 B apart, 8-dim groups
    128 B apart; LBO steps along K, SBO along M)."""
    rng = np.random.default_rng(K + N)
    a = rng.integers(-128, 128, size=(128, K)).astype(np.int8)
    b = rng.integers(-128, 128, size=(N, K)).astype(np.int8)
    ref = a.astype(np.int64) @ b.astype(np.int64).T
    assert np.array_equal(_i8_gemm(a, b, 0), ref)
    assert np.array_equal(_i8_gemm(a, b, 1), ref)
