"""bench.py's rank logic on the CPU: `--gpus 2` re-launches itself under torch.distributed.run,
two gloo ranks each run their shard of the streams through a stub engine, the device times are
max-reduced and the per-stream results gathered (the path's only collective); and the reference arm
reports the same workload config while mapping only the oracle library."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def last_json(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def run(*args, timeout=600):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    return last_json(p.stdout)


def test_two_rank_dry_run_gathers_every_stream():
    line = run("--dry-run", "--gpus", "2", "--config", "4", "--window", "2", "--steps", "2", "--warmup", "1")
    assert line["n_gpus"] == 2 and line["dry_run"]
    assert line["config"]["streams"] == 4 and line["config"]["streams_per_gpu"] == 2
    assert line["gather"]["streams"] == 4 and "gloo" in line["gather"]["via"]
    assert line["ms_per_rank_max"] > 0 and line["value"] > 0


def test_single_rank_dry_run_matches_gather_checksum():
    one = run("--dry-run", "--config", "4", "--window", "2", "--steps", "2", "--warmup", "1")
    two = run("--dry-run", "--gpus", "2", "--config", "4", "--window", "2", "--steps", "2", "--warmup", "1")
    assert one["gather"]["streams"] == two["gather"]["streams"] == 4
    assert abs(one["gather"]["checksum"] - two["gather"]["checksum"]) <= 1e-9 * abs(one["gather"]["checksum"])


def test_reference_arm_config_and_libraries():
    sys.path.insert(0, ROOT)
    import bench

    line = run("--impl", "reference", "--config", "0", "--steps", "1", "--warmup", "0", "--cpu-seconds", "1")
    assert line["impl"] == "reference"
    assert line["config"] == bench.workload(0, "full", 1)[0]
    assert line["libraries_mapped"] and all(p.startswith("oracle/") for p in line["libraries_mapped"]), line
