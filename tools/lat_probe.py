"""Lag-0 (window 1) per-line latency on configs[0]: wall of K back-to-back lines (device events) vs the
sum of the five kernels' own event times, to size the launch gaps."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2408_14947_b200 as pkg

spec = pkg.gen_spec(0)
x, _ = pkg.gen_lines(spec, 0, 64, want_mask=False)
P, B = 384, 108
dev = torch.from_numpy(x).cuda()
raw = torch.empty((1, P), dtype=torch.float32, device="cuda"); norm = torch.empty_like(raw)
for mode in ("full", "srp"):
    eng = pkg.Engine(pkg.ErxConfig(no_srp=mode == "full"), B, 1, 1)
    for k in range(5):
        eng.run_device(dev[k].data_ptr(), 1, P, raw.data_ptr(), norm.data_ptr(), first_index=k)
    eng.sync()
    K = 50
    eng.event_record(0)
    for k in range(K):
        eng.run_device(dev[k % 64].data_ptr(), 1, P, raw.data_ptr(), norm.data_ptr(), first_index=5 + k)
    eng.event_record(1)
    ms = eng.event_elapsed_ms(0, 1); eng.sync()
    eng.set_profiling(True)
    for k in range(K):
        eng.run_device(dev[k % 64].data_ptr(), 1, P, raw.data_ptr(), norm.data_ptr(), first_index=5 + K + k)
    eng.sync()
    kt = eng.kernel_times()
    tot = sum(v[0] for v in kt.values())
    print(mode, "wall ms/line", round(ms / K, 4), "kernels ms/line", round(tot / K, 4),
          {k: round(v[0] / max(v[1], 1), 4) for k, v in kt.items()})
    eng.close()
