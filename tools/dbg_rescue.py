"""Which windows of a full configs[4] run need the fp64 rescue, per factor kernel."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2408_14947_b200 as pkg  # noqa: E402

cid, T, n = 4, 32, int(sys.argv[1]) if len(sys.argv) > 1 else 3000
specs = [pkg.gen_spec(cid, s) for s in range(4)]
print("scene changes", [pkg.gen_scene_changes(sp) for sp in specs])
P, B = specs[0].pixels, specs[0].bands
for fac in (31, 30):
    eng = pkg.Engine(pkg.ErxConfig(no_srp=True, alpha=0.05), B, n_streams=4, window_lines=T)
    eng.set_factor_precision(fac)
    x = torch.empty((4, T, P, B), dtype=torch.float32, device="cuda")
    raw = torch.empty((4, T, P), dtype=torch.float32, device="cuda")
    norm = torch.empty_like(raw)
    last = 0
    hits = []
    for w0 in range(0, n - T + 1, T):
        for s in range(4):
            pkg.gen_lines_device(specs[s], w0, T, out=x[s], want_mask=False)
        torch.cuda.synchronize()
        eng.run_device(x.data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=w0)
        r = eng.rescued_lines()
        if r != last:
            hits.append((w0, r - last))
            last = r
    print("factor", eng.factor_precision(), "rescued", last, "windows", hits)
