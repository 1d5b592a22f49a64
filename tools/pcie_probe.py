"""Host<->device copy bandwidth from pinned memory (the e2e bound) and the e2e push/pop split."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

n = 283115520
h = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
el = (time.perf_counter() - t) / 5
print(f"H2D pinned {n / el / 1e9:.1f} GB/s ({el * 1e3:.2f} ms per 283 MB)")
t = time.perf_counter()
for _ in range(5):
    h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
el = (time.perf_counter() - t) / 5
print(f"D2H pinned {n / el / 1e9:.1f} GB/s")

import paper_2408_14947_b200 as pkg

S, T, P, B = 64, 16, 640, 108
x = np.stack([pkg.gen_lines(pkg.gen_spec(3, s), 0, T)[0] for s in range(S)])
pin = torch.from_numpy(x).pin_memory().numpy()
eng = pkg.Engine(pkg.ErxConfig(no_srp=True, alpha=0.1), B, n_streams=S, window_lines=T)
out = (np.empty((S, T, P)), np.empty((S, T, P)))
for k in range(3):
    eng.push(pin, k * T)
    eng.pop(out=out)
tp = tq = 0.0
for k in range(8):
    t0 = time.perf_counter()
    eng.push(pin, (k + 3) * T)
    t1 = time.perf_counter()
    eng.pop(out=out)
    t2 = time.perf_counter()
    tp += t1 - t0
    tq += t2 - t1
print(f"push {tp / 8 * 1e3:.2f} ms, pop {tq / 8 * 1e3:.2f} ms per 1024 lines -> {1024 / ((tp + tq) / 8):.0f} lines/s")
