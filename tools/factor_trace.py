"""Per-step timeline of one factor_blk CTA (an ERX_X_TRACE build of k_factor.cu):
  tools/ab_build.sh ftr "-DERX_X_TRACE" k_factor; ERX_B200_LIB=ab/ftr.so python tools/factor_trace.py
Events per thread: 1 step start, 2 panel done, 3 after the panel barrier, 4 trailing done, 5/6 diagonal
factor start / end (group 0), 7 sweep done, 8 planes written."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_14947_b200 as pkg  # noqa: E402
from paper_2408_14947_b200 import _lib  # noqa: E402

config, S, T = bench.workload(3, "full", 1, 0)
P, B = config["pixels"], config["bands"]
host = bench.build_pool(pkg, 3, list(range(S)), 2 * T)
dev = torch.from_numpy(host).cuda().view(S, 2, T, P, B).permute(1, 0, 2, 3, 4).contiguous()
raw = torch.empty((S, T, P), dtype=torch.float32, device="cuda")
norm = torch.empty_like(raw)
eng = pkg.Engine(pkg.ErxConfig(no_srp=True, alpha=config["alpha"]), B, S, T)
eng.set_graphs(False)
lib = C.CDLL(_lib.LIB_PATH)
buf = (C.c_ulonglong * (2 * 8192))()
for k in range(3):
    eng.run_device(dev[k % 2].data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=k * T)
eng.sync()
lib.erx_x_ftrace(buf, 8192)
eng.run_device(dev[1].data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=3 * T)
eng.sync()
n = lib.erx_x_ftrace(buf, 8192)
a = np.frombuffer(buf, dtype=np.uint64, count=2 * n).reshape(n, 2)
ev = [(int(t), int(v) >> 24, (int(v) >> 12) & 0xfff, int(v) & 0xfff) for t, v in a]
t0 = min(e[0] for e in ev)
print("events", n, "span cycles", max(e[0] for e in ev) - t0)
steps = sorted(set(e[2] for e in ev if e[1] in (1, 2, 3, 4)))
print(" k   start   panel(max thr)  bar1   trailing(min..max thr)  bar2   diag(start..end)")
for k in steps:
    if k < 2:
        continue
    def ts(i):
        return [e[0] - t0 for e in ev if e[1] == i and e[2] == k]
    s1, s2, s3, s4, s5, s6 = ts(1), ts(2), ts(3), ts(4), ts(5), ts(6)
    print(f"{k:2d} {min(s1):7d} {max(s2) - min(s1):7d} {max(s3) - max(s2):6d} "
          f"{min(s4) - max(s3):6d}..{max(s4) - max(s3):6d} "
          f"{(min(ts(1) if False else s4) if False else 0):1d}"
          f" diag {((min(s5) - max(s3)) if s5 else -1):6d}..{((max(s6) - max(s3)) if s6 else -1):6d}")
def last(i):
    v = [e[0] - t0 for e in ev if e[1] == i]
    return max(v) if v else None
def first(i):
    v = [e[0] - t0 for e in ev if e[1] == i]
    return min(v) if v else None
print("kernel start", first(9), "sweep start", first(0), "sweep done", last(7), "planes written", last(8))
