"""Diagnose the tcgen05 fp32 accumulation: signed relative error of the
6-product bf16x3 GEMM on all-positive data (bias shows up as a mean offset)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_14947_b200 import probe  # noqa: E402

for K in (16, 64, 256):
    for lo, hi in ((0.5, 1.0), (-1.0, 1.0)):
        rng = np.random.default_rng(K)
        a = rng.uniform(lo, hi, size=(128, K)).astype(np.float32)
        b = rng.uniform(lo, hi, size=(128, K)).astype(np.float32)
        ref = a.astype(np.float64) @ b.astype(np.float64).T
        da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        for split in (1,):
            dd = torch.zeros((128, 128), dtype=torch.float32, device="cuda")
            probe.lib().erx_tc_selftest(0, None, C.c_void_p(da.data_ptr()), C.c_void_p(db.data_ptr()), K, split,
                                        C.c_void_p(dd.data_ptr()))
            d = dd.cpu().numpy().astype(np.float64)
            # fp32-rounded exact result for comparison
            rel = (d - ref) / np.abs(ref).max()
            f32 = (ref.astype(np.float32).astype(np.float64) - ref) / np.abs(ref).max()
            print(f"K={K:3d} data[{lo},{hi}] split={split} mean_rel={rel.mean():+.3e} "
                  f"rms_rel={np.sqrt((rel**2).mean()):.3e} max={np.abs(rel).max():.3e} "
                  f"(fp32 rounding rms {np.sqrt((f32**2).mean()):.1e})")
