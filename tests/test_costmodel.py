"""Pins of the App. D replica-time cost model (oracle/costmodel.py) and the C++ ABI
lobra_replica_time against it (CPU)."""
import json
import os

import numpy as np
import pytest

from oracle import costmodel as CM

GOLD = os.path.join(os.path.dirname(__file__), "golden", "pp_cost_examples.json")
TS = {"b*s": lambda b, s: float(b * s), "unit": lambda b, s: 1.0 if b > 0 else 0.0,
      "b*s*s/16": lambda b, s: b * s * s / 16.0}


@pytest.mark.parametrize("case", json.load(open(GOLD))["cases"], ids=lambda c: c["name"])
def test_worked_examples(case):
    got = CM.replica_time(case["d"], case["s"], case["M"], TS[case["t"]], case["pp"])
    assert got == case["expect"], case["why"]


def test_pp1_is_the_no_pp_equation():
    """p = 1: the bubble vanishes, T = sum_j m_j t(b_j, s_j) + t(r_j, s_j)."""
    rng = np.random.default_rng(0)
    t = CM.quadratic_t(0.3, 1e-3, 2e-7)
    for _ in range(200):
        R = int(rng.integers(1, 8))
        s = sorted(int(x) for x in rng.integers(16, 4096, R))
        M = 8192
        d = [int(x) for x in rng.integers(0, 40, R)]
        want = 0.0
        for dj, sj in zip(d, s):
            bj = M // sj
            want += (dj // bj) * t(bj, sj) + t(dj % bj, sj)
        assert CM.replica_time(d, s, M, t, 1) == pytest.approx(want, rel=1e-15)


def test_fixed_length_pp_reduces_to_the_paper_equation():
    """One bucket, d = m b exactly (no remainder): T = m t(b, s) + (p - 1) t(b, s), the
    fixed-length 1F1B equation with micro-batch size b = mini-batch / m."""
    t = CM.quadratic_t(0.5, 2e-3, 1e-7)
    for p in (1, 2, 4, 8):
        for s in (128, 1024, 4096):
            M = 16384
            b = M // s
            for m in (1, 3, 7):
                got = CM.replica_time([m * b], [s], M, t, p)
                assert got == pytest.approx(CM.fixed_length_time(m * b, s, m, t, p), rel=1e-12)


def test_bubble_is_p_minus_1_times_the_longest_existing_chunk():
    """Reading Q29: only chunks that exist enter the max; adding empty buckets changes nothing."""
    t = CM.quadratic_t(0.0, 1.0, 0.0)
    base = CM.replica_time([3, 1], [2048, 512], 8192, t, 4)
    with_empty = CM.replica_time([3, 0, 1, 0], [2048, 4096, 512, 8192], 8192, t, 4)
    assert base == with_empty
    # bucket 2048: b = 4, m = 0, r = 3 -> remainder chunk t = 6144; bucket 512: r = 1 -> 512
    assert base == pytest.approx(6144 + 512 + 3 * 6144)


def test_linear_in_full_chunks():
    """With t proportional to b (c0 = 0, c2 = 0) and remainders included, the compute term is
    exactly sum_j d_j t(1, s_j): App. D's linearity in d."""
    t = CM.quadratic_t(0.0, 3e-3, 0.0)
    d, s = [37, 5, 120], [3000, 700, 64]
    got = CM.replica_time(d, s, 8192, t, 1)
    assert got == pytest.approx(sum(dj * t(1, sj) for dj, sj in zip(d, s)), rel=1e-12)


def test_cpp_matches_oracle():
    from paper_2509_01193_b200 import _lib
    rng = np.random.default_rng(3)
    for _ in range(300):
        R = int(rng.integers(1, 10))
        s = [int(x) for x in rng.integers(1, 8192, R)]
        d = [int(x) for x in rng.integers(0, 60, R)]
        c = (float(rng.uniform(0, 1)), float(rng.uniform(0, 1e-3)), float(rng.uniform(0, 1e-7)))
        p = int(rng.integers(1, 9))
        want = CM.replica_time(d, s, 8192, CM.quadratic_t(*c), p)
        got = _lib.lobra_replica_time(d, s, 8192, p, *c)
        assert got == pytest.approx(want, rel=1e-12, abs=1e-12)


def test_cpp_rejects_bad_input():
    from paper_2509_01193_b200 import _lib
    for d, s, M, p in (([1], [10], 8, 1), ([-1], [4], 8, 1), ([1], [4], 8, 0), ([1], [0], 8, 1)):
        with pytest.raises(_lib.LobraError):
            _lib.lobra_replica_time(d, s, M, p, 1.0, 1.0, 0.0)
