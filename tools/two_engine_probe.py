"""Two engines, each with half of the streams, on their own CUDA streams (cross-window overlap between the
halves) against one engine with all streams:  python tools/two_engine_probe.py [config] [mode] [window] [steps]"""
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_14947_b200 as pkg  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
mode = sys.argv[2] if len(sys.argv) > 2 else "full"
config, S, T = bench.workload(cid, mode, 1, int(sys.argv[3]) if len(sys.argv) > 3 else 0)
K = int(sys.argv[4]) if len(sys.argv) > 4 else 20
NE = int(os.environ.get("ENGINES", "2"))
P, B = config["pixels"], config["bands"]
n_win = max(2, math.ceil(2 * bench.L2_BYTES / (S * T * P * B * 4)))
host = bench.build_pool(pkg, cid, list(range(S)), n_win * T)
dev = torch.from_numpy(host).cuda().view(S, n_win, T, P, B).permute(1, 0, 2, 3, 4).contiguous()  # [win][S][T][P][B]
raw = torch.empty((S, T, P), dtype=torch.float32, device="cuda")
norm = torch.empty_like(raw)
Sh = S // NE
engs = [pkg.Engine(pkg.ErxConfig(no_srp=mode == "full", alpha=config["alpha"]), B, Sh, T) for _ in range(NE)]


def step(k):
    w = dev[k % n_win]
    for i, e in enumerate(engs):
        e.run_device(w[i * Sh:(i + 1) * Sh].data_ptr(), T, P, raw[i * Sh:(i + 1) * Sh].data_ptr(),
                     norm[i * Sh:(i + 1) * Sh].data_ptr(), first_index=k * T)


for k in range(3):
    step(k)
for e in engs:
    e.sync()
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(3, 3 + K):
    step(k)
for e in engs:
    e.sync()
ms = (time.perf_counter() - t0) * 1e3 / K
print(f"{NE} engine(s) x {Sh} streams, c{cid} {mode} T={T}: {ms:.4f} ms/step (wall), {S * T / ms * 1e3 / 1e6:.3f} M lines/s")
