"""Per-line error of the engine vs the oracle on the edge cases, for each factor precision / stats kind."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import oracle_ctypes as orc  # noqa: E402
import paper_2408_14947_b200 as pkg  # noqa: E402
from test_gpu_numerics import structured_lines  # noqa: E402
from test_gpu_parity import ocfg  # noqa: E402


def case_dn(B, noise, L=12):
    rng = np.random.default_rng(int(B + 1e6 * noise))
    P = 640
    A = rng.normal(0, 0.05, size=(B, 3))
    base = 0.3 + 0.2 * np.sin(np.linspace(0, 3, B))
    x = ((base + rng.normal(size=(40, P, 3)) @ A.T + rng.normal(0, noise, size=(40, P, B))) * 3000.0)
    return x.astype(np.float32)[:L]


def run(cfg, x, factor=None, stats=None, window=4):
    L_, P, B = x.shape
    eng = pkg.Engine(cfg, B, window_lines=window)
    if factor is not None:
        eng.set_factor_precision(factor)
    if stats is not None:
        eng.set_stats_tensor(stats)
    eng.push(x[None], 0)
    eng.finish()
    _, _, raw, _ = eng.pop()
    info = (eng.stats_tensor(), eng.factor_precision(), eng.kernel_times() if False else None)
    eng.close()
    return raw[0], info


def report(label, cfg, x):
    raw_o, _, _ = orc.run_stream(ocfg(orc, cfg), x)
    for factor in (0, 64, 1):
        for stats in (2, 0):
            try:
                raw_g, info = run(cfg, x, factor, stats)
            except Exception as ex:
                print(label, factor, stats, "ERR", ex)
                continue
            rel = np.abs(raw_g - raw_o) / np.abs(raw_o)
            per = " ".join(f"{np.median(r):.1e}" for r in rel[:8])
            print(f"{label} factor={factor}->{info[1]} stats={stats}->{info[0]}: max {rel.max():.2e} med {np.median(rel):.2e} | per-line med {per}")


cfg = pkg.ErxConfig(no_srp=True, alpha=0.1, buffer_len=0)
report("DN108 1e-3", cfg, case_dn(108, 1e-3))
report("DN124 5e-5", cfg, case_dn(124, 5e-5))
report("DN12 2e-4", cfg, case_dn(12, 2e-4))
rng = np.random.default_rng(24)
report("P2 B24", pkg.ErxConfig(no_srp=True, alpha=0.5, buffer_len=0), structured_lines(rng, 16, 2, 24))
rng = np.random.default_rng(260)
report("P100 B160", cfg, structured_lines(rng, 24, 100, 160))
