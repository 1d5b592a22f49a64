"""Timeline of CTA 0 of the warp-specialised statistics kernel (an ERX_X_TRACE build):
  tools/ab_build.sh tr "-DERX_X_TRACE" k_stats_i8; ERX_STATS_WS=3 ERX_B200_LIB=ab/tr.so python tools/stats_trace.py"""
import ctypes as C
import math
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
if os.environ.get("ERX_STATS_ONEPASS"):
    eng.set_stats_onepass(int(os.environ["ERX_STATS_ONEPASS"]))
lib = C.CDLL(_lib.LIB_PATH)
lib.erx_x_trace.restype = C.c_int
buf = (C.c_ulonglong * (2 * 32768))()
for k in range(3):
    eng.run_device(dev[k % 2].data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=k * T)
eng.sync()
lib.erx_x_trace(buf, 32768)
eng.run_device(dev[1].data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=3 * T)
eng.sync()
n = lib.erx_x_trace(buf, 32768)
a = np.frombuffer(buf, dtype=np.uint64, count=2 * n).reshape(n, 2)
a = a[np.argsort(a[:, 0])]
t0 = int(a[0, 0])
names = {6: "Q range", 7: "Q quant-done", 8: "Q tmem-read", 0: "Q sready", 1: "Q full2", 2: "Q pempty", 3: "Q planes", 4: "Q accfull", 5: "Q epi-done",
         10: "R full1", 11: "R sready", 20: "M pfull", 21: "M commit", 30: "P1 issue", 31: "P2 issue"}
lines = [(int(t) - t0, int(v) >> 24, (int(v) >> 12) & 0xfff, int(v) & 0xfff) for t, v in a]
kmax = max(l[2] for l in lines)
print("events", n, "lines", kmax + 1, "span cycles", lines[-1][0])
for kk in (kmax // 2, kmax // 2 + 1):
    sel = [l for l in lines if l[2] == kk]
    print(f"--- line {kk}")
    for t, i, k, c in sel:
        print(f"{t:9d} {names.get(i, i):12s} c={c}")
# per-line durations
starts = {}
for t, i, k, c in lines:
    if i == 0 or (i == 1 and c == 0): starts[k] = t
print("line starts (Q sready):", [starts.get(k) for k in range(kmax + 1)])
