cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_tc_selftest.py -q -x -p no:cacheprovider 2>&1 | tail -15
timeout 300 python - <<'PY'
import ctypes as C, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2408_14947_b200 as pkg
eng = pkg.Engine(pkg.ErxConfig(no_srp=True), 8)
rng = np.random.default_rng(0)
a = rng.integers(-128, 128, size=(128, 64)).astype(np.int8); b = rng.integers(-128, 128, size=(112, 64)).astype(np.int8)
ref = a.astype(np.int64) @ b.astype(np.int64).T
for (lbo, sbo) in ((128, 512), (512, 128)):
    da = torch.from_numpy(a).cuda(); db = torch.from_numpy(b).cuda(); dd = torch.zeros((128, 112), dtype=torch.int32, device='cuda')
    st = pkg.lib().erx_tc_selftest_i8(eng._h, C.c_void_p(da.data_ptr()), C.c_void_p(db.data_ptr()), 64, 112, 1, 512, 128, lbo, sbo, C.c_void_p(dd.data_ptr()))
    d = dd.cpu().numpy().astype(np.int64)
    print('lbo', lbo, 'sbo', sbo, 'status', st, 'exact', np.array_equal(d, ref), 'maxerr', np.abs(d - ref).max())
PY
