"""Full-length parity fixtures: the fp64 CPU oracle over whole BASELINE streams.

The oracle needs minutes per stream at D = B (configs[1]: 10,000 lines x
68 MFLOP; configs[4]: 3,000 lines x 544 MFLOP), too slow for the GPU test
budget, so it runs here once and the GPU tests (tests/test_gpu_fullstream.py)
compare against what it leaves in tests/golden/full_<case>.npz:

  samp_lines   [n_samp]           sampled line indices (every 100th line, plus the lines
                                  right after each scene change)
  raw, norm    [S][n_samp][P]     oracle raw delta and norm on those lines (float32)
  top_idx      [m]                flat indices into the pooled non-warmup norm scores
                                  (stream-major, then line, then pixel) of the oracle's
                                  top 1.25 %, ordered by descending norm
  top_val      [m]                their oracle norm (float32)
  k            ()                 top-1 % size, ceil(0.01 * pooled)
  auc          ()                 oracle roc_auc of the pooled non-warmup norm vs the labels
  meta                            json: config id, streams, lines, mode, alpha, window

Inputs come from the same seeded generator the GPU tests use (erx_gen_lines /
its device twin, bit-identical), so only scores are stored.  Run:

    python tests/golden/make_full_fixtures.py [case ...]     (all cases: ~15 min on 8 cores)
"""
import json
import math
import os
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

# case: (config id, streams, lines, no_srp, alpha, GPU window)
CASES = {
    "c3_dB": (3, (0, 31, 63), 5000, True, 0.1, 32),
    "c3_d5": (3, (0, 31, 63), 5000, False, 0.1, 32),
    "c1_dB": (1, (0,), 10000, True, 0.05, 256),
    "c1_d5": (1, (0,), 10000, False, 0.05, 256),
    "c4_dB": (4, (0,), 3000, True, 0.05, 32),
    "c4_d5": (4, (0,), 3000, False, 0.05, 32),
}
BUFFER = 99
TOP_FRAC, KEEP_FRAC = 0.01, 0.0125


def sample_lines(n, scene):
    s = set(range(50, n, 100))
    for c in scene:
        if 0 < c < n:
            s.update(c + d for d in (0, 1, 2, 5, 10, 20) if c + d < n)
    return np.array(sorted(s), np.int64)


def scene_lines(orc, spec):
    return orc.gen_scene_changes(spec)


def run_stream(pkg, orc, cid, s, n, no_srp, alpha, samp, log):
    spec = pkg.gen_spec(cid, s)
    cfg = orc.OracleConfig(no_srp=no_srp, alpha=alpha, buffer_len=BUFFER)
    det = orc.OracleErx(cfg, spec.bands)
    P = spec.pixels
    raw_s = np.zeros((samp.size, P), np.float32)
    norm_s = np.zeros((samp.size, P), np.float32)
    pooled = np.zeros((n - BUFFER, P), np.float64)
    labels = np.zeros((n - BUFFER, P), np.uint8)
    where = {int(t): i for i, t in enumerate(samp)}
    t0 = time.time()
    for c0 in range(0, n, 100):
        m = min(100, n - c0)
        x, mask = pkg.gen_lines(spec, c0, m, threads=1)
        for u in range(m):
            t = c0 + u
            raw, norm, _ = det.process(t, x[u])
            if t in where:
                raw_s[where[t]] = raw
                norm_s[where[t]] = norm
            if t >= BUFFER:
                pooled[t - BUFFER] = norm
                labels[t - BUFFER] = mask[u]
        if c0 % 1000 == 0:
            log(f"c{cid} s{s} {'D=B' if no_srp else 'd=5'}: line {c0 + m}/{n} ({time.time() - t0:.0f} s)")
    return raw_s, norm_s, pooled.ravel(), labels.ravel()


def make_case(name, pkg, orc, pool, log):
    cid, streams, n, no_srp, alpha, window = CASES[name]
    spec0 = pkg.gen_spec(cid, streams[0])
    scene = sorted({c for s in streams for c in scene_lines(pkg, pkg.gen_spec(cid, s))})
    samp = sample_lines(n, scene)
    futs = [pool.submit(run_stream, pkg, orc, cid, s, n, no_srp, alpha, samp, log) for s in streams]
    res = [f.result() for f in futs]
    raw = np.stack([r[0] for r in res])
    norm = np.stack([r[1] for r in res])
    pooled = np.concatenate([r[2] for r in res])
    labels = np.concatenate([r[3] for r in res])
    k = int(math.ceil(TOP_FRAC * pooled.size))
    m = int(math.ceil(KEEP_FRAC * pooled.size))
    part = np.argpartition(-pooled, m - 1)[:m]
    order = part[np.argsort(-pooled[part], kind="stable")]
    auc = orc.roc_auc(pooled, labels)
    meta = dict(case=name, config=cid, streams=list(streams), lines=n, no_srp=no_srp, alpha=alpha,
                buffer_len=BUFFER, window=window, pixels=spec0.pixels, bands=spec0.bands, scene_changes=scene,
                generator="erx_gen_lines (include/erx_datagen.h), BASELINE.json configs[%d]" % cid,
                made_by="tests/golden/make_full_fixtures.py")
    out = os.path.join(HERE, f"full_{name}.npz")
    np.savez_compressed(out, samp_lines=samp, raw=raw, norm=norm, top_idx=order.astype(np.uint32),
                        top_val=pooled[order].astype(np.float32), k=np.int64(k), auc=np.float64(auc),
                        meta=np.array(json.dumps(meta)))
    log(f"wrote {out}: pooled {pooled.size}, k {k}, auc {auc:.6f}, {os.path.getsize(out) / 1e6:.2f} MB")


def main():
    import oracle_ctypes as orc

    names = sys.argv[1:] or list(CASES)
    lock = threading.Lock()

    def log(msg):
        with lock:
            print(msg, flush=True)

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 8) as pool:
        outer = ThreadPoolExecutor(max_workers=len(names))
        fs = [outer.submit(make_case, nm, orc, orc, pool, log) for nm in names]
        for f in fs:
            f.result()
        outer.shutdown()


if __name__ == "__main__":
    main()
