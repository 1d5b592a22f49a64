"""Run two configs[3]-shaped windows (and two configs[0] windows) and save raw / norm, for a bitwise
A/B of two builds or of kernel variants selected by environment (e.g. ERX_STATS_WS=0 vs 3):
  ERX_STATS_WS=0 python tools/ab_bitwise.py out0.npz; python tools/ab_bitwise.py out1.npz out0.npz"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_14947_b200 as pkg  # noqa: E402

out = {}
for cid, S, T in ((3, 16, 32), (0, 1, 16)):
    cfg = bench.CONFIGS[cid]
    P, B = cfg["pixels"], cfg["bands"]
    host = bench.build_pool(pkg, cid, list(range(S)), 2 * T)
    dev = torch.from_numpy(host).cuda().view(S, 2, T, P, B).permute(1, 0, 2, 3, 4).contiguous()
    raw = torch.empty((S, T, P), dtype=torch.float32, device="cuda")
    norm = torch.empty_like(raw)
    eng = pkg.Engine(pkg.ErxConfig(no_srp=True, alpha=cfg["alpha"]), B, S, T)
    for w in range(2):
        eng.run_device(dev[w].data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=w * T)
        eng.sync()
        out[f"c{cid}_raw{w}"] = raw.cpu().numpy().copy()
        out[f"c{cid}_norm{w}"] = norm.cpu().numpy().copy()
    eng.close()
np.savez(sys.argv[1], **out)
if len(sys.argv) > 2:
    ref = np.load(sys.argv[2])
    for k in out:
        same = np.array_equal(out[k], ref[k])
        print(k, "bitwise equal" if same else f"DIFF max {np.nanmax(np.abs(out[k] - ref[k])):.3e}")
