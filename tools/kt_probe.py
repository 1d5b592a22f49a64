"""Per-kernel device times (engine profiling events) of one bench workload, for A/B builds:
  ERX_B200_LIB=path/to/lib.so python tools/kt_probe.py [config] [mode] [window] [steps]"""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_14947_b200 as pkg  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
mode = sys.argv[2] if len(sys.argv) > 2 else "full"
config, S, T = bench.workload(cid, mode, 1, int(sys.argv[3]) if len(sys.argv) > 3 else 0)
K = int(sys.argv[4]) if len(sys.argv) > 4 else 20
P, B = config["pixels"], config["bands"]
n_win = max(2, math.ceil(2 * bench.L2_BYTES / (S * T * P * B * 4)))
host = bench.build_pool(pkg, cid, list(range(S)), n_win * T)
dev = torch.from_numpy(host).cuda().view(S, n_win, T, P, B).permute(1, 0, 2, 3, 4).contiguous()
raw = torch.empty((S, T, P), dtype=torch.float32, device="cuda")
norm = torch.empty_like(raw)
eng = pkg.Engine(pkg.ErxConfig(no_srp=mode == "full", alpha=config["alpha"]), B, S, T)
if os.environ.get("ERX_FACTOR"):
    eng.set_factor_precision(int(os.environ["ERX_FACTOR"]))
if os.environ.get("ERX_STATS_ONEPASS"):
    eng.set_stats_onepass(int(os.environ["ERX_STATS_ONEPASS"]))
if os.environ.get("ERX_DEVICE_GROUPS"):
    eng.set_device_groups(int(os.environ["ERX_DEVICE_GROUPS"]))
if os.environ.get("ERX_FACTOR_THREADS"):
    eng.set_factor_threads(int(os.environ["ERX_FACTOR_THREADS"]))
for k in range(3):
    eng.run_device(dev[k % n_win].data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=k * T)
eng.sync()
eng.event_record(0)
for k in range(3, 3 + K):
    eng.run_device(dev[k % n_win].data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=k * T)
eng.event_record(1)
ms = eng.event_elapsed_ms(0, 1) / K
eng.set_profiling(True)
for k in range(K):
    eng.run_device(dev[k % n_win].data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=k * T)
eng.sync()
kt = eng.kernel_times()
print(os.environ.get("ERX_B200_LIB", "default"), f"factor={eng.factor_precision()}", f"redone={eng.stats_redone_lines()}", f"c{cid} {mode} T={T}: {ms:.4f} ms/step, {S * T / ms * 1e3 / 1e6:.3f} M lines/s |",
      " ".join(f"{k} {v[0] / max(v[1], 1):.4f}" for k, v in kt.items()))
