"""factor_blk CTA size on a configs[1] (D = 224) or configs[0] (D = 108, lag 0) window: per-launch factor
time from the engine's event timing, for each ERX_OPT_FACTOR_THREADS value."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_14947_b200 as pkg

for cid, T in ((1, 256), (0, 1), (0, 32)):
    spec = pkg.gen_spec(cid)
    x, _ = pkg.gen_lines(spec, 0, 4 * T, want_mask=False)
    P, B = x.shape[1], x.shape[2]
    dev = torch.from_numpy(x).cuda()
    raw = torch.empty((T, P), dtype=torch.float32, device="cuda"); norm = torch.empty_like(raw)
    for th in (128, 256):  # (a 512-thread variant measured 0.254 vs 0.189 ms on configs[1]: not kept)
        eng = pkg.Engine(pkg.ErxConfig(no_srp=True, alpha=0.1), B, 1, T)
        eng.set_factor_threads(th)
        for k in range(2):
            eng.run_device(dev[k * T].data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=k * T)
        eng.sync()
        eng.set_profiling(True)
        for k in range(2, 4):
            eng.run_device(dev[k * T].data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=k * T)
        eng.sync()
        kt = eng.kernel_times()
        print(f"c{cid} T={T} threads={th} factor ms/launch {kt['factor'][0] / max(kt['factor'][1], 1):.4f}")
        eng.close()
