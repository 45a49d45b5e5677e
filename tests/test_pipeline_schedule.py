"""Host logic of the PP (1F1B) executor (paper_2509_01193_b200/pipeline.py; SURVEY NEXT-3,
App. D): the per-stage op order, its dependency-respecting simulation, and
the textbook 1F1B makespan (m + p - 1)(t_f + t_b) for equal micro-batches."""
import itertools

import numpy as np
import pytest

from paper_2509_01193_b200.pipeline import schedule_1f1b, simulate_1f1b


@pytest.mark.parametrize("p,m", list(itertools.product([1, 2, 3, 4, 8], [1, 2, 3, 5, 8, 16])))
def test_schedule_shape(p, m):
    for s in range(p):
        ops = schedule_1f1b(p, s, m)
        assert sorted(k for o, k in ops if o == "F") == list(range(m))
        assert [k for o, k in ops if o == "B"] == list(range(m))      # backwards in order
        inflight, peak = 0, 0
        seen_f = set()
        for o, k in ops:
            if o == "F":
                seen_f.add(k)
                inflight += 1
            else:
                assert k in seen_f                                   # F_k before B_k
                inflight -= 1
            peak = max(peak, inflight)
        assert peak <= min(p - s, m)                                 # activation memory bound


@pytest.mark.parametrize("p,m", [(1, 4), (2, 4), (4, 4), (4, 8), (8, 16), (3, 7)])
def test_equal_microbatches_textbook_makespan(p, m):
    tf, tb = 1.0, 2.0
    assert simulate_1f1b(p, [tf] * m, [tb] * m) == pytest.approx((m + p - 1) * (tf + tb))


def test_variable_microbatches_bubble_bound():
    """Variable-length micro-batches in the order lobra_dispatch emits them (descending cost,
    SURVEY §8(c) c2 step 9): the makespan lies between one stage's work and that work plus
    (p - 1) times the largest micro-batch -- App. D's bubble term -- and the
    upper bound is attained.  (In an arbitrary order 1F1B can exceed it several times over:
    the ordering is what makes App. D's model hold.)"""
    rng = np.random.default_rng(0)
    tight = 0.0
    for _ in range(300):
        p = int(rng.integers(2, 6))
        m = int(rng.integers(1, 12))
        tf = np.sort(rng.uniform(0.2, 3.0, m))[::-1]
        tb = 2 * tf
        t = simulate_1f1b(p, list(tf), list(tb))
        work = float(np.sum(tf + tb))
        bound = (p - 1) * float(np.max(tf + tb))
        assert work - 1e-9 <= t <= work + bound + 1e-9
        tight = max(tight, (t - work) / bound)
    assert tight > 0.999
