"""Pins the oracle's had::Rng / mix_seed / ErrorKind restatement against
golden vectors produced by the reference's own rng.hpp / errors.hpp
(tests/golden/ref_golden.json, made by tests/golden/make_golden.py)."""
import json
import os

import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ref_golden.json")))
SEEDS = [0, 1, 42, 0xDEADBEEF]


@pytest.mark.parametrize("seed", SEEDS)
def test_rng_streams(oracle, seed):
    r = oracle.Rng(seed)
    assert [str(r.next_u64()) for _ in range(16)] == GOLD[f"next_u64_seed{seed}"]
    r = oracle.Rng(seed)
    assert [r.uniform() for _ in range(16)] == GOLD[f"uniform_seed{seed}"]
    r = oracle.Rng(seed)
    assert [float(r.uniform_f32()) for _ in range(16)] == GOLD[f"uniform_f32_seed{seed}"]
    r = oracle.Rng(seed)
    got = [r.normal() for _ in range(17)]
    # Box-Muller goes through libm log/sin/cos: allow 1 ulp-scale slack.
    for g, w in zip(got, GOLD[f"normal_seed{seed}"]):
        assert g == pytest.approx(w, rel=1e-15, abs=1e-15)
    r = oracle.Rng(seed)
    bounds = [1, 2, 3, 7, 10, 100, 1000003, 0x8000000000000001]
    got = [str(r.below(b)) for _ in range(2) for b in bounds]
    assert got == GOLD[f"below_seed{seed}"]
    r = oracle.Rng(seed)
    assert [str(i) for i in r.sample_indices(50, 12)] == GOLD[f"sample_indices_50_12_seed{seed}"]
    r = oracle.Rng(seed)
    mix = []
    for _ in range(6):
        mix.append(r.normal())
        mix.append(r.uniform())
    for g, w in zip(mix, GOLD[f"normal_uniform_mix_seed{seed}"]):
        assert g == pytest.approx(w, rel=1e-15, abs=1e-15)


def test_mix_seed(oracle):
    got = [str(oracle.mix_seed(s, n)) for s in SEEDS for n in (0, 1, 2, 99, 5000, 0xFFFFFFFFFFFFFFFF)]
    assert got == GOLD["mix_seed"]


def test_error_kinds_match_reference():
    # The C-ABI status codes (include/erx_b200.h) are the reference ErrorKind values.
    assert GOLD["error_kinds"] == {"config": 2, "data": 3, "metric_undefined": 4, "numeric": 5, "io": 6}
    assert GOLD["exit_codes"]["config"] == 2 and GOLD["exit_codes"]["data"] == 3
    assert GOLD["exit_codes"]["numeric"] == 3 and GOLD["factorization_pivot"] == 7
