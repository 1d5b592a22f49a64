"""Tiny workloads covering every kernel of the path, for compute-sanitizer (one tool per run):
  compute-sanitizer --tool racecheck python tools/sanitize_run.py
Exercises: stats_i8 + c0 fold + scan + factor_blk (int8 W planes) + score_i8 + normalize + fixup (configs[3]
lines, 2 streams); the chunked scan + small path (configs[2], one stream, 64-line window); the FFMA stats /
score + factor_blk (224 bands); factor_cl (448 bands, cluster) and factor_big; the fp64 rescue
(an ill-conditioned radiance-scale line); the host (pinned, grouped) path."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2408_14947_b200 as pkg  # noqa: E402


def run(cid, S, n, T, no_srp=True, factor=0, P=None, x=None, alpha=None):
    specs = [pkg.gen_spec(cid, s) for s in range(S)]
    if x is None:
        x = np.stack([pkg.gen_lines(sp, 0, n)[0] for sp in specs])
        if P:
            x = np.ascontiguousarray(x[:, :, :P])
    B = x.shape[3]
    cfg = pkg.ErxConfig(no_srp=no_srp, alpha=alpha or 0.1, buffer_len=1)
    eng = pkg.Engine(cfg, B, n_streams=S, window_lines=T)
    eng.set_factor_precision(factor)
    eng.push(x, 0)
    eng.finish()
    idx, _, raw, _ = eng.pop()
    assert idx.size == n and np.isfinite(raw).all()
    print(f"c{cid} S={S} n={n} T={T} D={'B' if no_srp else 'd'} factor={eng.factor_precision()} "
          f"stats={eng.stats_tensor()} rescued={eng.rescued_lines()} ok", flush=True)
    eng.close()


run(3, 2, 6, 3, P=160)                 # tensor path (stats_i8 / score_i8 / factor_blk planes)
run(3, 2, 6, 3, no_srp=False, P=160)   # d = 5 SRP small path
run(2, 1, 70, 64, P=256)               # chunked scan, identity small path
run(1, 1, 4, 2, P=96)                  # FFMA stats / score, factor_blk at 224 bands
run(4, 1, 2, 1, P=64, factor=30)       # thread-block-cluster factor
run(4, 1, 2, 1, P=64, factor=31)       # factor_big
rng = np.random.default_rng(0)
A = rng.normal(0, 0.05, size=(40, 3))
dn = ((0.3 + rng.normal(size=(1, 3, 200, 3)) @ A.T + rng.normal(0, 2e-4, size=(1, 3, 200, 40))) * 3000.0)
run(3, 1, 3, 3, x=dn.astype(np.float32))  # ill-conditioned: the fp64 rescue
print("sanitize workloads done")
