"""The C++ header mirror (include/erx_b200/hadkit_b200.hpp) compiles against
the C ABI with reference-style code, and (on a GPU) runs the line-scan loop."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_hadkit_mirror.cpp")
LIBDIR = os.path.join(ROOT, "paper_2408_14947_b200")


def build(tmp_path):
    exe = str(tmp_path / "test_hadkit_mirror")
    subprocess.run(["make", "-s", "-C", os.path.join(LIBDIR, "csrc")], check=True)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
                    "-L", LIBDIR, "-l:liberx_b200.so", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_cpp_mirror_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_cpp_mirror_runs_line_scan_loop(tmp_path):
    out = subprocess.run([build(tmp_path)], check=True, capture_output=True, text=True).stdout
    f = json.loads(out.strip().splitlines()[-2])  # the reference's free functions through the mirror
    assert f["normalize_err"] < 1e-5 and f["srp_weights_match"] and f["ema_fixed"] and f["identity_ok"]
    assert (f["z_rows"], f["z_cols"], f["stats_d"]) == (384, 5, 5) and f["threshold"] == [0, 0, 1]
    assert f["srp_lines"] == 5
    r = json.loads(out.strip().splitlines()[-1])
    assert r["lines"] == 40 and r["order_ok"] and r["name"] == "erx" and r["warmup0"]
    assert abs(r["norm_mean"]) < 1e-5 and r["lines_seen"] == 40 and r["dims"] == 108
    assert r["config_exit"] == 2 and r["data_exit"] == 3 and r["numeric_kind"] == 5 and r["pivot"] >= 0
