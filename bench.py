#!/usr/bin/env python3
"""ERX hot-path benchmark (driver contract: one JSON line from rank 0).

Workload (default): BASELINE.json configs[3] — 64 independent scan streams,
P=640 pixels x B=108 bands, alpha=0.1, full covariance (D = B, no_srp),
streams sharded evenly over the ranks (no data-path collective).  One step =
one window of T lines of every local stream through the five-kernel
pipeline (stats -> scan -> factor -> score -> normalize) on inputs already
resident in HBM.  Lines come from the BASELINE generator and are replayed
from a device pool at least 2x the L2 size, so no step reads inputs left in
L2 by the previous one.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 3] [--mode full|srp] [--window T]

`--gpus N` without a torchrun environment re-launches itself under
`torch.distributed.run` with N ranks (one per GPU, NCCL, 127.0.0.1); each rank
scores its shard of the streams, the device times are max-reduced and the
per-stream results are gathered to rank 0 (the path's only collective).
`--dry-run` runs the same rank / timing / gather logic with a CPU stub engine
over gloo (tests/test_bench_ranks.py).

`--impl reference` times the fp64 CPU restatement of the reference path
(oracle/, "port": the reference ships declarations only) on the host cores; it
maps only the oracle library (which carries its own copy of the seeded
generator), never a product library.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    0: dict(streams=1, pixels=384, bands=108, alpha=0.1, lines=2000),
    1: dict(streams=1, pixels=640, bands=224, alpha=0.05, lines=10000),
    2: dict(streams=1, pixels=1024, bands=10, alpha=0.1, lines=20000),
    3: dict(streams=64, pixels=640, bands=108, alpha=0.1, lines=5000),
    4: dict(streams=4, pixels=1280, bands=448, alpha=0.05, lines=3000),
}
L2_BYTES = 126 * 1024 * 1024


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


LINES_PER_GPU_WINDOW = 4096


def workload(cid, mode, world, window=0):
    """The benchmark workload of BASELINE.json configs[cid] at `world` ranks: (config dict shared by both
    arms, streams per rank, window T).  The window (lag per stream) defaults to ~4096 lines per GPU
    (T = 64 at N = 1, 512 at N = 8) so each GPU's launches stay full as the fixed streams spread out
    (measured on configs[3] D = B at N = 1: T = 32 / 48 / 64 / 96 -> 3.45 / 3.56 / 3.65 / 3.72 M lines/s;
    a window of >= 1024 lines runs as two stream groups of half the streams on two CUDA streams)."""
    cfgd = CONFIGS[cid]
    S_tot = cfgd["streams"]
    S = max(1, S_tot // world)
    # (the d = 5 path's windows are cheap -- 0.22 ms per 4096 lines -- so its fixed per-window costs weigh
    # more: 8192 lines per GPU, measured 18.3 -> 19.5 M lines/s on configs[3])
    per_gpu = LINES_PER_GPU_WINDOW * (2 if mode == "srp" else 1)
    T = window if window else min(max(32, per_gpu // S), cfgd["lines"] // 2)
    no_srp = mode == "full"
    config = {"workload": f"configs[{cid}]", "streams": S_tot, "streams_per_gpu": S, "pixels": cfgd["pixels"],
              "bands": cfgd["bands"], "dims": cfgd["bands"] if no_srp else 5,
              "mode": "D=B (no_srp)" if no_srp else "d=5 SRP", "alpha": cfgd["alpha"], "window_lines": T,
              "lines_per_stream": cfgd["lines"],
              "l2": "inputs larger than L2: device pool >= 2x L2, one window per step"}
    return config, S, T


def free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args):
    """--gpus N outside torchrun: re-exec under torch.distributed.run with N ranks on this node."""
    env = dict(os.environ)
    if not args.dry_run:
        env.setdefault("NCCL_DEBUG", "INFO")  # the communicator's rank count shows in the log
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


class StubEngine:
    """--dry-run: the engine's step / timing surface on the CPU (a fixed per-line reduction), so the
    rank, timing and gather logic of run_ours runs over gloo without a GPU."""

    def __init__(self, S, T, P, B):
        self.S, self.T, self.P = S, T, P
        self.raw = np.zeros((S, T, P))
        self.t = [0.0] * 8
        self.launches = 0

    def run_device(self, x, k):
        self.raw = x.sum(axis=-1, dtype=np.float64) + k  # [S][T][P]
        self.launches += 5

    def event_record(self, slot):
        self.t[slot] = time.perf_counter()

    def event_elapsed_ms(self, a, b):
        return (self.t[b] - self.t[a]) * 1e3


NCU_SUMMARY = os.path.join(ROOT, "profiles", "r02j_ncu_full_c3.txt")  # one group of 4096 lines per launch (T = 64)
NCU_NAMES = {"stats": ("stats_i8_ws_kernel", "stats_i8_kernel", "stats_kernel", "stats_small"),
             "score": ("score_i8_kernel", "score_kernel"), "factor": ("factor_blk_kernel",),
             "scan": ("scan_tile_kernel", "scan_kernel"), "normalize": ("normalize_kernel",)}


def ncu_traffic(kernel):
    """DRAM bytes per launch (read + write) of `kernel` from the committed ncu --set full summary
    (tools/ncu_summary.py output), or None when it has no entry for it."""
    try:
        text = open(NCU_SUMMARY).read()
    except OSError:
        return None
    for block in text.split("== ")[1:]:
        name = block.split("\n", 1)[0]
        if not any(n in name for n in NCU_NAMES.get(kernel, ())):
            continue
        vals = {}
        for line in block.splitlines()[1:]:
            parts = line.split()
            if len(parts) >= 3 and parts[0] in ("dram_read", "dram_write"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(parts[2], None)
                if scale:
                    vals[parts[0]] = float(parts[1]) * scale
        if len(vals) == 2:
            return {"bytes": vals["dram_read"] + vals["dram_write"],
                    "source": os.path.relpath(NCU_SUMMARY, ROOT) + f" ({name.strip()}, one launch, ncu --set full)"}
    return None


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int, enabled: bool = True):
        self.device = device
        self.proc = None
        self.enabled = enabled

    def __enter__(self):
        if not self.enabled:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return False
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            out = ""
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)
        return False

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def algorithmic(cfgd, D, srp_nnz=0):
    """Per-line algorithmic work: bytes read/written and flops per kernel."""
    P, B = cfgd["pixels"], cfgd["bands"]
    tri = D * (D + 1)  # 2 * D(D+1)/2 (flops of a symmetric rank-1 update / a triangular matvec per pixel)
    proj = 2 * P * srp_nnz
    return {
        "bytes_line": 4 * P * B + 8 * P,
        "flops_line": 2 * P * D * D + D ** 3 / 3 + proj,
        "stats": dict(flops=P * tri + proj, bytes=4 * P * B),
        "score": dict(flops=P * tri + proj, bytes=4 * P * B + 4 * P),
        # factor: Cholesky + triangular inverse; reads the packed fp64 prior, writes packed fp32 W blocks
        "factor": dict(flops=2 * D ** 3 / 3, bytes=8 * D * (D + 1) // 2 + 4 * 64 * ((D + 7) // 8) * ((D + 15) // 8) // 2),
        # scan: reads [c | s | S] and writes the pre-update (mu, K) per line, fp64
        "scan": dict(flops=0, bytes=8 * (2 * D + D * (D + 1) // 2) + 8 * (D + D * (D + 1) // 2)),
        "normalize": dict(flops=0, bytes=8 * P),
        "fixup": dict(flops=0, bytes=0),  # fp64 rescue: no listed lines on the BASELINE configs
    }


def build_pool(pkg, cid, streams, lines_per_stream, threads=0):
    """[S][L][P][B] fp32 host pool from the BASELINE generator."""
    out = []
    for s in streams:
        x, _ = pkg.gen_lines(pkg.gen_spec(cid, s), 0, lines_per_stream, threads=threads, want_mask=False)
        out.append(x)
    return np.stack(out)


def run_ours(args):
    rank, world, local = dist_env()
    dry = args.dry_run
    if not dry:
        import torch

        import paper_2408_14947_b200 as pkg

        torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo" if dry else "nccl")
    cid = args.config
    cfgd = CONFIGS[cid]
    from paper_2408_14947_b200.sharding import gather_stream_results, max_over_ranks, shard_streams

    S_tot = cfgd["streams"]
    if S_tot % world:
        raise SystemExit(f"{S_tot} streams do not shard evenly over {world} ranks")
    shard_n = args.shard_of if (args.shard_of and world == 1) else world  # --shard-of: one rank's share on 1 GPU
    my_streams = list(shard_streams(S_tot, shard_n, 0 if shard_n != world else rank))
    config, S, T = workload(cid, args.mode, shard_n, args.window)
    assert S == len(my_streams)
    P, B = cfgd["pixels"], cfgd["bands"]
    no_srp = args.mode == "full"
    line_bytes = P * B * 4
    dev_str = "cpu" if dry else f"cuda:{local}"
    if dry:  # a small CPU pool of the real generator's lines (the oracle library's copy of it)
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle_ctypes as orc

        n_win = 2
        pool_lines = n_win * T
        t0 = time.time()
        host = build_pool(orc, cid, my_streams, pool_lines, threads=1)
        gen_s = time.time() - t0
        dev = host.reshape(S, n_win, T, P, B).transpose(1, 0, 2, 3, 4).copy()
        eng = StubEngine(S, T, P, B)
        D = B if no_srp else 5

        def step(k):
            eng.run_device(dev[k % n_win], k)
    else:
        n_win = max(2, math.ceil(2 * L2_BYTES / (S * T * line_bytes)))
        pool_lines = n_win * T
        t0 = time.time()
        host = build_pool(pkg, cid, my_streams, pool_lines)
        gen_s = time.time() - t0
        dev = torch.from_numpy(host).to(dev_str)
        # windows laid out [win][S][T][P][B] so each step reads one contiguous block
        dev = dev.view(S, n_win, T, P, B).permute(1, 0, 2, 3, 4).contiguous()
        raw = torch.empty((S, T, P), dtype=torch.float32, device=dev_str)
        norm = torch.empty_like(raw)
        cfg = pkg.ErxConfig(no_srp=no_srp, alpha=cfgd["alpha"])
        eng = pkg.Engine(cfg, B, n_streams=S, window_lines=T, device=local)
        eng.set_factor_precision(args.factor)
        eng.set_stats_tensor(args.stats)
        D = eng.dims

        def step(k):
            w = k % n_win
            eng.run_device(dev[w].data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=k * T)

    def sync():
        if not dry:
            eng.sync()
            torch.cuda.synchronize()

    for k in range(args.warmup):
        step(k)
    sync()
    if dist:
        dist.barrier()
    launches0 = eng.launches if dry else eng.launch_count()
    with ClockSampler(local, enabled=not dry) as clk:
        eng.event_record(0)
        for k in range(args.steps):
            step(args.warmup + k)
        eng.event_record(1)
        ms = eng.event_elapsed_ms(0, 1)
    sync()
    launches = (eng.launches if dry else eng.launch_count()) - launches0
    ms_max = max_over_ranks(ms, dist, device=dev_str)
    lines_total = S * world * T * args.steps  # = S_tot * T * steps (one rank's share with --shard-of)
    value = lines_total / (ms_max / 1e3)
    # the final gather (the path's only collective): per-stream results of the last window to every
    # rank, checked complete on rank 0 (here the fp64 sum of each stream's raw scores)
    last = eng.raw if dry else raw.double().sum(dim=(1, 2)).cpu().numpy()
    local_res = {sid: np.array([float(np.sum(last[i]))]) for i, sid in enumerate(my_streams)}
    if shard_n != world:  # --shard-of: the other ranks' shares are not run
        gathered = {"streams": len(my_streams), "note": f"rank 0 share of {shard_n} only"}
    else:
        allres = gather_stream_results(local_res, S_tot, dist)
        gathered = {"streams": len(allres), "checksum": float(sum(float(a[0]) for a in allres)),
                    "via": ("all_gather_object over " + ("gloo" if dry else "NCCL")) if dist else "local"}
    if dry:
        if rank == 0:
            line = {"metric": "lines/sec (batched independent streams, aggregate over GPUs)", "value": value,
                    "unit": "lines/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                    "ms_per_step": ms_max / args.steps, "ms_per_rank_max": ms_max, "higher_is_better": True,
                    "scaling": "strong", "vs_baseline": None, "dry_run": True, "config": config,
                    "gather": gathered, "gpu_launches": 0, "gen_seconds": gen_s,
                    "data": "synthetic: BASELINE.json generator; CPU stub engine (no kernels)"}
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        if rank == 0:
            print(json.dumps(line), flush=True)
        return

    # per-kernel device time (CUDA events on the engine stream), separate pass
    eng.set_profiling(True)
    prof_steps = max(3, min(args.steps, 10))
    for k in range(prof_steps):
        step(k)
    eng.sync()
    kt = eng.kernel_times()
    eng.set_profiling(False)
    alg = algorithmic(cfgd, D)
    total_k = sum(v[0] for v in kt.values()) or 1.0
    kernels = {}
    for name, (kms, cnt) in kt.items():
        per = kms / max(cnt, 1)
        lines_per_launch = S * T
        a = alg[name]
        kernels[name] = {"ms_per_launch": per, "share": kms / total_k, "launches": cnt,
                         "tflops": a["flops"] * lines_per_launch / (per * 1e-3) / 1e12 if per > 0 and a["flops"] else None,
                         "gbs": a["bytes"] * lines_per_launch / (per * 1e-3) / 1e9 if per > 0 and a["bytes"] else None}
    dom = max(kernels, key=lambda k: kernels[k]["share"])
    from paper_2408_14947_b200 import probe

    reg_peak, const_peak = probe.fp32_tflops(local, eng.cuda_stream)
    fp32_peak = max(reg_peak, const_peak)  # the larger (conservative) measured FFMA rate
    fprec = eng.factor_precision()
    pk = peaks()
    dk = kernels[dom]
    src = (f"measured FFMA probe on this GPU in this run (erx_probe_fp32_tflops: register-form "
           f"{reg_peak:.1f}, constant-form {const_peak:.1f} TFLOP/s; the larger is the peak)")
    tensor = eng.stats_tensor() == 2
    if dom in ("stats", "score") and tensor:
        # exact-integer tcgen05 kernels stream the line from HBM (the digit-plane MMAs are not the
        # algorithmic flops): the bound is the line's bytes at the measured HBM bandwidth
        roof = {"bound": "hbm", "kernel": dom, "achieved": dk["gbs"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": dk["gbs"] / pk["hbm_gbs"] if dk["gbs"] else None, "traffic": None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "algorithmic": f"{alg[dom]['bytes']} B/line x {S*T} lines/launch"}
    elif alg[dom]["flops"] > 0 and dom in ("stats", "score") and no_srp:
        roof = {"bound": "fp32", "kernel": dom, "achieved": dk["tflops"], "peak": fp32_peak, "unit": "TFLOP/s",
                "frac": dk["tflops"] / fp32_peak, "traffic": None, "peak_source": src,
                "algorithmic": f"{alg[dom]['flops']:.4g} flop/line x {S*T} lines/launch"}
    elif alg[dom]["flops"] > 0 and dom == "factor":
        fpk = fp32_peak if fprec == 32 else fp32_peak / 2
        roof = {"bound": "fp32" if fprec == 32 else "fp64", "kernel": dom, "achieved": dk["tflops"], "peak": fpk,
                "unit": "TFLOP/s", "frac": dk["tflops"] / fpk, "traffic": None,
                "peak_source": src + ("" if fprec == 32 else "; fp64 = half (B200 FP64:FP32 = 1:2)"),
                "algorithmic": f"{alg[dom]['flops']:.4g} flop/line x {S*T} lines/launch"}
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": dk["gbs"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": dk["gbs"] / pk["hbm_gbs"] if dk["gbs"] else None, "traffic": None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "algorithmic": f"{alg[dom]['bytes']} B/line x {S*T} lines/launch"}
    tr = ncu_traffic(dom)
    if tr:
        roof["traffic"] = tr["bytes"]
        roof["traffic_source"] = tr["source"]
        roof["algorithmic_bytes"] = alg[dom]["bytes"] * S * T
    # whole-pipeline roofline per the north star: slower of flops@peak and bytes@HBM per line
    t_flop = alg["flops_line"] / (fp32_peak * 1e12)
    t_byte = alg["bytes_line"] / (pk["hbm_gbs"] * 1e9)
    roof_lines = 1.0 / max(t_flop, t_byte)
    roofline_line = {"lines_per_s_roofline_per_gpu": roof_lines, "bound": "fp32" if t_flop > t_byte else "hbm",
                     "frac": (value / world) / roof_lines,
                     "lines_per_s_hbm_bound_per_gpu": 1.0 / t_byte, "frac_of_hbm_bound": (value / world) * t_byte,
                     "note": "fp32 bound = 2 P D^2 + D^3/3 flop/line at the measured FFMA peak; hbm bound = "
                             "4 P B + 8 P bytes/line (read the line, write raw+norm) at MEASURED_PEAKS hbm_gbs"}

    # end-to-end through the public C ABI with HOST buffers (pinned), H2D + D2H inside the timed region
    e2e = None
    try:
        e2e_steps = max(2, min(args.steps, 8))
        eng2 = pkg.Engine(cfg, B, n_streams=S, window_lines=T, device=local)
        eng2.set_factor_precision(args.factor)
        eng2.set_host_groups(args.host_groups)
        eng2.set_stats_tensor(args.stats)
        eng2.set_async_host(not args.sync_host)
        pin = torch.from_numpy(np.ascontiguousarray(host[:, :T])).pin_memory().numpy()
        outb = (np.empty((S, T, P)), np.empty((S, T, P)))  # caller-owned ScoredLine payload buffers
        popped = 0
        for k in range(2):
            eng2.push(pin, k * T)
            eng2.pop(out=outb)
        eng2.finish()
        while eng2.ready():
            eng2.pop(out=outb)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for k in range(e2e_steps):
            # pipelined: this window's copy-in overlaps the previous window's kernels and result
            # copies; pop returns the previous window's ScoredLine payload
            eng2.push(pin, (k + 2) * T)
            popped += eng2.pop(out=outb)[0].size
        eng2.finish()
        while eng2.ready():
            popped += eng2.pop(out=outb)[0].size
        el = time.perf_counter() - t0
        assert popped == T * e2e_steps, (popped, T * e2e_steps)
        el_t = torch.tensor([el], dtype=torch.float64, device=f"cuda:{local}")
        if dist:
            dist.all_reduce(el_t, op=dist.ReduceOp.MAX)
        e2e = {"value": S * world * T * e2e_steps / float(el_t.item()), "unit": "lines/s",
               "h2d_bytes_per_step": S * T * P * B * 4, "d2h_bytes_per_step": S * T * (P * 4 * 2 + 4),
               "path": "erx_push_host (pinned) -> 6 kernels -> erx_pop (fp64 ScoredLine payload)",
               "pipelined": not args.sync_host}
        eng2.close()
        # the e2e path's own bound: the line's bytes over the measured pinned host->device bandwidth
        pc = pcie_bandwidth(local)
        e2e["pcie"] = pc
        if pc.get("h2d_gbs"):
            bound = pc["h2d_gbs"] * 1e9 / (P * B * 4)  # lines/s per GPU the H2D copy alone allows
            e2e["pcie_bound_lines_per_s"] = bound * world
            e2e["frac_of_pcie_bound"] = e2e["value"] / (bound * world)
    except Exception as ex:  # report, never hide
        e2e = {"error": repr(ex)}

    extra = {}
    if world == 1 and not args.quick:
        extra = secondary_measurements(pkg, args)
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cid, no_srp, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": "lines/sec (batched independent streams, aggregate over GPUs)",
            "value": value, "unit": "lines/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": ("f32 input; stats+score exact int8-digit tcgen05 (s32 TMEM), f32 factor, f64 scan/state"
                      if tensor else "f32 (FFMA stats/whitening) + f64 (scan, Cholesky, inverse)"),
            "data": f"synthetic: BASELINE.json configs[{cid}] generator (include/erx_datagen.h), device pool >= 2x L2 replayed",
            "config": config,
            "engine": {"factor_precision": eng.factor_precision(), "stats_kernel": "tcgen05 kind::i8" if tensor
                       else "FFMA", "pool_lines_per_stream": pool_lines, "dims": D,
                       "rescued_lines": eng.rescued_lines(),
                       "shard": f"rank 0 share of {args.shard_of} GPUs" if shard_n != world else "own"},
            "gather": gathered,
            "pixel_bands_per_s": value * P * B,
            "roofline": roof, "roofline_line": roofline_line, "kernels": kernels,
            "e2e": e2e, "clocks": clk.summary(), "gpu_launches": int(launches),
            "cpu_baseline": cpu, "gen_seconds": gen_s,
        }
        line.update(extra)
    if dist:  # tear the communicator down first: NCCL's own log lines must not follow the JSON line
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        sys.stdout.flush()
        print(json.dumps(line), flush=True)


def secondary_measurements(pkg, args):
    """Side numbers named by the metric (1 GPU): single-stream throughput on configs[1] and
    configs[2], the batched configs[3] workload with the reference's default d = 5 projection, the
    batched configs[4] (448 bands) workload, and configs[0] lag-0 per-line latency (north-star
    target < 1 ms at 108 bands)."""
    import torch

    out = {}

    def throughput(cid, T, modes, streams=(0,), K=20, factor=0):
        """lines/s of a device-resident window of T lines per stream (inputs cycled through a pool
        >= 2x L2), per mode; also per-line HBM traffic vs the measured peak (4PB + 8P bytes/line) and
        the per-kernel device times of a separate profiled pass."""
        cfgd = CONFIGS[cid]
        P, B = cfgd["pixels"], cfgd["bands"]
        S = len(streams)
        n_win = max(2, math.ceil(2 * L2_BYTES / (S * T * P * B * 4)))
        host = build_pool(pkg, cid, list(streams), n_win * T)
        dev = torch.from_numpy(host).cuda().view(S, n_win, T, P, B).permute(1, 0, 2, 3, 4).contiguous()
        raw = torch.empty((S, T, P), dtype=torch.float32, device="cuda")
        norm = torch.empty_like(raw)
        res = {}
        for mode in modes:
            eng = pkg.Engine(pkg.ErxConfig(no_srp=mode == "full", alpha=cfgd["alpha"]), B, S, T)
            eng.set_factor_precision(factor)
            for k in range(3):
                eng.run_device(dev[k % n_win].data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=k * T)
            eng.sync()
            eng.event_record(0)
            for k in range(3, 3 + K):
                eng.run_device(dev[k % n_win].data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=k * T)
            eng.event_record(1)
            ms = eng.event_elapsed_ms(0, 1)
            eng.sync()
            lps = K * S * T / (ms / 1e3)
            gbs = lps * (4 * P * B + 8 * P) / 1e9
            eng.set_profiling(True)
            for k in range(3):
                eng.run_device(dev[k % n_win].data_ptr(), T, P, raw.data_ptr(), norm.data_ptr(), first_index=k * T)
            eng.sync()
            kt = {kk: round(v[0] / max(v[1], 1), 5) for kk, v in eng.kernel_times().items()}
            res[mode] = {"lines_per_s": lps, "pixel_bands_per_s": lps * P * B, "hbm_gbs_algorithmic": gbs,
                         "hbm_frac": gbs / peaks()["hbm_gbs"], "factor_kernel": eng.factor_precision(),
                         "kernel_ms_per_window": kt}
            eng.close()
        del dev
        return res

    try:
        # a single stream only parallelises across the lines of a window: use a deep lag
        out["single_stream"] = {"workload": "configs[1]: 1 stream, 640 px x 224 bands, alpha=0.05",
                                "window_lines": 256, **throughput(1, 256, ("full", "srp"))}
    except Exception as ex:
        out["single_stream"] = {"error": repr(ex)}
    try:
        # the same stream at a deeper lag (1024 lines, ~10 % of the stream): the per-line factor of one
        # stream only fills the GPU with enough lines per window
        out["single_stream_deep"] = {"workload": "configs[1]: 1 stream, 640 px x 224 bands, alpha=0.05",
                                     "window_lines": 1024, **throughput(1, 1024, ("full",), K=10)}
    except Exception as ex:
        out["single_stream_deep"] = {"error": repr(ex)}
    try:
        out["single_stream_c2"] = {"workload": "configs[2]: 1 stream, 1024 px x 10 bands, alpha=0.1",
                                   "window_lines": 2048, **throughput(2, 2048, ("full", "srp"))}
    except Exception as ex:
        out["single_stream_c2"] = {"error": repr(ex)}
    try:
        t_srp = workload(3, "srp", 1)[2]  # the headline's window (~4096 lines per GPU)
        out["batched_srp"] = {"workload": "configs[3] with the reference default d = 5 SRP: 64 streams, "
                                          "640 px x 108 bands, alpha=0.1", "window_lines": t_srp,
                              **throughput(3, t_srp, ("srp",), streams=tuple(range(64)))}
    except Exception as ex:
        out["batched_srp"] = {"error": repr(ex)}
    try:
        out["batched_c4"] = {"workload": "configs[4]: 4 streams, 1280 px x 448 bands, alpha=0.05, D = B",
                             "window_lines": 32, **throughput(4, 32, ("full",), streams=(0, 1, 2, 3), K=10)}
        out["batched_c4_deep"] = {"workload": "configs[4]: 4 streams, 1280 px x 448 bands, alpha=0.05, D = B",
                                  "window_lines": 128, **throughput(4, 128, ("full",), streams=(0, 1, 2, 3), K=4)}
        # the same window with the thread-block-cluster factor (DSMEM, 4 CTAs per line) forced
        out["batched_c4_cluster_factor"] = {"workload": "as batched_c4, ERX_OPT_FACTOR_PRECISION = 30",
                                            **throughput(4, 32, ("full",), streams=(0, 1, 2, 3), K=5, factor=30)}
        # lag 0 at 448 bands: one stream, one line per window (the cluster kernel's regime) vs factor_big
        lat4 = {}
        for fac, name in ((0, "auto"), (31, "factor_big")):
            r = throughput(4, 1, ("full",), streams=(0,), K=20, factor=fac)["full"]
            lat4[name] = {"ms_per_line": 1e3 / r["lines_per_s"], "factor_kernel": r["factor_kernel"],
                          "kernel_ms_per_window": r["kernel_ms_per_window"]}
        out["latency_c4"] = {"workload": "configs[4] stream 0: 1280 px x 448 bands, window = 1 (no lag)", **lat4}
    except Exception as ex:
        out["batched_c4"] = {"error": repr(ex)}
    try:
        cfgd = CONFIGS[0]
        P, B = cfgd["pixels"], cfgd["bands"]
        host = build_pool(pkg, 0, [0], 64)
        dev = torch.from_numpy(host[0]).cuda()
        raw = torch.empty((1, P), dtype=torch.float32, device="cuda")
        norm = torch.empty_like(raw)
        lat = {}
        for mode in ("full", "srp"):
            for graphs in (True, False):
                eng = pkg.Engine(pkg.ErxConfig(no_srp=mode == "full"), B, 1, 1)
                eng.set_graphs(graphs)
                # the caller streams lines through a 4-slot device ring (the graph cache holds 8 windows)
                for k in range(8):
                    eng.run_device(dev[k % 4].data_ptr(), 1, P, raw.data_ptr(), norm.data_ptr())
                eng.sync()
                K = 64
                eng.event_record(0)
                for k in range(K):
                    eng.run_device(dev[k % 4].data_ptr(), 1, P, raw.data_ptr(), norm.data_ptr())
                eng.event_record(1)
                ms = eng.event_elapsed_ms(0, 1)
                eng.sync()
                lat[mode + ("" if graphs else "_no_graph")] = {"ms_per_line": ms / K}
                eng.close()
        out["latency"] = {"workload": "configs[0]: 384 px x 108 bands, window=1 (no lag), device-resident, "
                                      "one CUDA-graph launch per line (and kernel-by-kernel for comparison)", **lat}
    except Exception as ex:
        out["latency"] = {"error": repr(ex)}
    try:
        out["dropin_single_stream"] = dropin_measurement()
    except Exception as ex:
        out["dropin_single_stream"] = {"error": repr(ex)}
    try:
        out["metrics"] = metrics_measurement(pkg)
    except Exception as ex:
        out["metrics"] = {"error": repr(ex)}
    try:
        out["datagen"] = datagen_measurement(pkg)
    except Exception as ex:
        out["datagen"] = {"error": repr(ex)}
    return out


def dropin_measurement(lines=2000):
    """The drop-in single-stream e2e number: configs[0] through the C++ had::ErxDetector::process
    (include/hadkit/erx.hpp -> C ABI) one host line per call, wall clock from the first line fed to
    the last ScoredLine (tools/dropin_bench.cpp), at lag 32 and lag 0."""
    import tempfile

    lib = os.path.join(ROOT, "paper_2408_14947_b200")
    exe = os.path.join(tempfile.mkdtemp(), "dropin_bench")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tools", "dropin_bench.cpp"), "-L", lib, "-l:liberx_b200.so",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    out = subprocess.run([exe, str(lines)], check=True, capture_output=True, text=True, timeout=600).stdout
    return json.loads(out.strip().splitlines()[-1])


def datagen_measurement(pkg):
    """The input generator on the device vs the host generator (all host
    threads): configs[3] lines of one stream, fp32 [n][640][108] + masks, CUDA events around
    erx_gen_lines_device (which returns synchronised)."""
    import torch

    spec = pkg.gen_spec(3, 0)
    n = 2048
    out = torch.empty((n, spec.pixels, spec.bands), dtype=torch.float32, device="cuda")
    mask = torch.empty((n, spec.pixels), dtype=torch.uint8, device="cuda")
    pkg.gen_lines_device(spec, 0, n, out, mask)  # warm-up (module load, scratch allocation)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    pkg.gen_lines_device(spec, 0, n, out, mask, stream=st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    m = 256
    t0 = time.perf_counter()
    xh, _ = pkg.gen_lines(spec, 0, m)
    el = time.perf_counter() - t0
    xd = out[:m].cpu().numpy()
    neq = int(np.count_nonzero(xd.view(np.int32) != xh.view(np.int32)))
    return {"workload": f"configs[3] stream 0, lines 0..{n - 1} (640 px x 108 bands)", "lines_per_s": n / (ms / 1e3),
            "gb_per_s_written": n * spec.pixels * spec.bands * 4 / (ms / 1e3) / 1e9,
            "ms": ms, "host_lines_per_s": m / el, "host_threads": os.cpu_count(),
            "values_differing_from_host": neq, "values_compared": int(xd.size)}


def metrics_measurement(pkg):
    """Parity-gate metrics on the device at the c3 pooled size: the exact
    tie-grouped ROC AUC and the top-1% set over 64 x (5000 - 99) x 640 non-warmup scores.
    Synthetic stand-in scores (N(0,1), anomalies +3, 0.3% labelled; ties from fp32 rounding),
    device-resident; CUDA events on the calling stream.  CPU reference: the oracle's roc_auc
    (std::sort + trapezoid, 1 thread) on a 2 M-score sample."""
    import torch
    from paper_2408_14947_b200 import metrics

    n = 64 * (5000 - 99) * 640
    g = torch.Generator(device="cuda").manual_seed(0)
    y = (torch.rand(n, device="cuda", generator=g) < 0.003).to(torch.uint8)
    s = torch.randn(n, device="cuda", generator=g) + 3.0 * y.float()
    st = torch.cuda.current_stream()
    k = int(math.ceil(0.01 * n))
    metrics.roc_auc(s, y, stream=st.cuda_stream)  # warm-up (allocator, module load)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record(st)
    auc = metrics.roc_auc(s, y, stream=st.cuda_stream)
    ev[1].record(st)
    mask, cut = metrics.top_k(s, k, stream=st.cuda_stream)
    ev[2].record(st)
    torch.cuda.synchronize()
    auc_ms, topk_ms = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    res = {"workload": "c3 pooled non-warmup scores: 64 x 4901 lines x 640 px (synthetic stand-in)",
           "scores": n, "auc": auc, "auc_ms": auc_ms, "auc_scores_per_s": n / (auc_ms / 1e3),
           "top1pct_ms": topk_ms, "top1pct_k": k,
           "algorithm": "4-pass 8-bit LSD radix sort (in-house kernels) + exact integer Mann-Whitney count"}
    try:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle_ctypes
        m = 2_000_000
        hs, hy = s[:m].double().cpu().numpy(), y[:m].cpu().numpy()
        t0 = time.perf_counter()
        oracle_ctypes.roc_auc(hs, hy)
        el = time.perf_counter() - t0
        res["cpu_baseline"] = {"value": m / el, "unit": "scores/s", "cores": 1, "kind": "port",
                               "sample": f"oracle roc_auc on the first {m} scores"}
    except Exception as ex:
        res["cpu_baseline"] = {"error": repr(ex)}
    return res


def cpu_baseline(cid, no_srp, seconds=12.0, threads=None):
    """fp64 oracle (port of the reference path) on a bounded sample of the same workload."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_ctypes as orc  # oracle library only: its own copy of the seeded generator, no product .so

    cfgd = CONFIGS[cid]
    cores = threads or os.cpu_count() or 1
    S = min(cfgd["streams"], cores) if cfgd["streams"] > 1 else 1
    use_threads = S
    ocfg = orc.OracleConfig(no_srp=no_srp, alpha=cfgd["alpha"])
    probe = build_pool(orc, cid, [0], 3)
    t0 = time.perf_counter()
    orc.run_streams(ocfg, probe, threads=1, want_scores=False)
    per_line = (time.perf_counter() - t0) / 3
    n_lines = int(max(4, min(cfgd["lines"], seconds / max(per_line, 1e-6))))
    pool = build_pool(orc, cid, list(range(S)), n_lines)
    t0 = time.perf_counter()
    orc.run_streams(ocfg, pool, threads=use_threads, want_scores=False)
    el = time.perf_counter() - t0
    lps = S * n_lines / el
    model = ""
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        pass
    return {"value": lps, "unit": "lines/s", "cores": use_threads, "kind": "port",
            "sample": f"{S} stream(s) x {n_lines} lines of configs[{cid}] ({'D=B' if no_srp else 'd=5'}), "
                      f"one stream per thread, {el:.1f} s wall", "cpu_model": model,
            "pixel_bands_per_s": lps * cfgd["pixels"] * cfgd["bands"]}


def run_reference(args):
    """The reference path on the host cores: the fp64 C++ restatement (oracle/erx_oracle.cpp, the
    reference ships declarations only) through its own C API, all host threads, one stream per thread;
    each step a bounded sample of the same workload.  Maps the oracle library only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cid = args.config
    no_srp = args.mode == "full"
    config, _, _ = workload(cid, args.mode, world, args.window)
    samples = []
    cores = os.cpu_count() or 1
    last = None
    for k in range(args.warmup + args.steps):
        r = cpu_baseline(cid, no_srp, seconds=args.cpu_seconds / max(1, args.steps + args.warmup) * 2, threads=cores)
        if k >= args.warmup:
            samples.append(r["value"])
        last = r
    value = float(np.mean(samples))
    line = {
        "impl": "reference", "metric": "lines/sec (batched independent streams, aggregate over GPUs)",
        "value": value, "unit": "lines/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: BASELINE.json configs[{cid}] generator (the oracle library's copy)",
        "config": config,
        "cpu_baseline": {"value": value, "unit": "lines/s", "cores": last["cores"], "kind": "port",
                         "sample": last["sample"], "cpu_model": last.get("cpu_model")},
        "e2e": {"value": value, "unit": "lines/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference ships headers only (no bodies, no Eigen); timed path is the fp64 C++ restatement "
                "oracle/erx_oracle.cpp through its own C API (naive scalar fp64, one stream per host thread)",
        "libraries_mapped": mapped_libraries(),
    }
    print(json.dumps(line), flush=True)


def mapped_libraries():
    """This repository's shared libraries mapped into the process (/proc/self/maps)."""
    out = set()
    try:
        for l in open("/proc/self/maps"):
            path = l.split()[-1]
            if path.startswith(ROOT) and ".so" in path:
                out.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(out)


def pcie_bandwidth(device, nbytes=256 << 20):
    """Pinned host <-> device copy bandwidth (GB/s, best of 5) on this GPU: the e2e path's own peak."""
    import torch

    try:
        h = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
        d = torch.empty(nbytes // 4, dtype=torch.float32, device=f"cuda:{device}")
        st = torch.cuda.current_stream(device)
        res = {}
        for name, fn in (("h2d_gbs", lambda: d.copy_(h, non_blocking=True)),
                         ("d2h_gbs", lambda: h.copy_(d, non_blocking=True))):
            best = 0.0
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                fn()
                e1.record(st)
                e1.synchronize()
                best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
            res[name] = best
        res["bytes"] = nbytes
        return res
    except Exception as ex:
        return {"error": repr(ex)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3, choices=[0, 1, 2, 3, 4])
    ap.add_argument("--mode", default="full", choices=["full", "srp"])
    ap.add_argument("--window", type=int, default=0, help="lines per stream per window (0: ~4096 lines per GPU)")
    ap.add_argument("--factor", type=int, default=0, choices=[0, 1, 32, 64],
                    help="factor kernel precision (ERX_OPT_FACTOR_PRECISION)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip the single-stream / latency side measurements")
    ap.add_argument("--stats", type=int, default=2, choices=[0, 2],
                    help="line-statistics / score kernels: 0 FFMA, 2 tcgen05 exact int8 digits")
    ap.add_argument("--host-groups", type=int, default=0, help="stream groups per host window (0 auto)")
    ap.add_argument("--shard-of", type=int, default=0,
                    help="N=1 only: run rank 0's stream share of an N-GPU job (value is per GPU)")
    ap.add_argument("--sync-host", action="store_true", help="e2e without ERX_OPT_ASYNC_HOST (push waits for scores)")
    ap.add_argument("--dry-run", action="store_true", help="CPU stub engine over gloo: rank / timing / gather logic only")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
