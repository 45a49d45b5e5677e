"""Pins of the integer dispatch oracle (SPEC/paper examples, brute force,
Eq. 3 constraints, the §3 worked instance).  CPU only."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import dispatch as D

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "dispatch_spec_examples.json")))


def test_histogram_example():
    g = GOLD["histogram"]
    assert D.histogram(g["lengths"], g["grid_step"], g["grid_max"]).tolist() == g["counts"]
    assert D.histogram([], 256, 512).tolist() == [0, 0]
    with pytest.raises(D.DispatchError):
        D.histogram([513], 256, 512)


@pytest.mark.parametrize("case", GOLD["dp"])
def test_dp_examples(case):
    b, pad = D.dynamic_buckets(np.array(case["counts"]), case["grid_step"], case["R"])
    assert b == case["boundaries"] and pad == case["padding"]


def test_padding_cost_example():
    g = GOLD["padding_cost"]
    assert D.padding_cost(g["lengths"], g["boundaries"]) == g["padding"]


def _brute_buckets(counts, step, R):
    occ = [k + 1 for k in range(len(counts)) if counts[k]]
    best = None
    for m in range(1, min(R, len(occ)) + 1):
        for sub in itertools.combinations(occ[:-1], m - 1):
            bl = [k * step for k in sub] + [occ[-1] * step]
            pad = 0
            for k in occ:
                u = k * step
                pad += counts[k - 1] * (min(s for s in bl if s >= u) - u)
            key = (pad, bl)
            if best is None or key < best:
                best = key
    return best[1], best[0]


def test_dp_equals_exhaustive_subsets():
    """DP optimality and the lexicographic tie-break vs exhaustive boundary subsets
    (S:223 [DERIVED])."""
    rng = np.random.default_rng(11)
    for _ in range(300):
        U = int(rng.integers(1, 10))
        counts = rng.integers(0, 4, size=U) * (rng.random(U) < 0.7)
        if counts.sum() == 0:
            counts[rng.integers(0, U)] = 1
        R = int(rng.integers(1, 5))
        got = D.dynamic_buckets(counts, 256, R)
        assert got == _brute_buckets(counts.tolist(), 256, R), (counts, R)


def test_dp_padding_reconstruction():
    """Total padding = State_{U,R} + intra-interval constant (P:617 footnote)."""
    rng = np.random.default_rng(12)
    for _ in range(50):
        lens = rng.integers(1, 2048, size=int(rng.integers(1, 60)))
        counts = D.histogram(lens, 256, 2048)
        R = int(rng.integers(1, 6))
        b, cross = D.dynamic_buckets(counts, 256, R)
        intra = sum(-(-int(l) // 256) * 256 - int(l) for l in lens)
        assert D.padding_cost(lens, b) == cross + intra


def test_split_and_microbatch_and_replica_time_examples():
    # split d=5, p=2 -> {3,2}; replica time with c = s: M=8, s=4, d=5 -> 20 ... on one
    # group with p=1 and one with p=2.
    g = GOLD["microbatch"]
    res = D.dispatch([D.Group(1, 1, g["M"])], [[4, 8]], [4] * g["count"], [0] * g["count"],
                     grid_step=4, grid_max=8, R=1)
    sizes = np.bincount(res.seq_chunk).tolist()
    assert sizes == g["chunks"]
    assert res.replica_cost.tolist() == [GOLD["replica_time"]["time"]]
    gs = GOLD["split"]
    res = D.dispatch([D.Group(1, gs["p"], 8)], [[4, 8]], [4] * gs["d"], [0] * gs["d"], 4, 8, 1)
    assert np.bincount(res.seq_replica).tolist() == gs["counts"]


def test_design_anatomy_instance():
    """§3 instance: n={1,2,4,8}, r={1,2,3,4}, B={196,62,16,4}, p={4,2,0,1}.
    Costs are not printed; use a cost that grows with length and shrinks with TP.  All
    Eq. 3 constraints hold, bucket 4 lands on the r=4 group, p=0 gets nothing."""
    g = GOLD["design_anatomy"]
    step = 256
    bl = [256, 512, 768, 1024]
    lens = sum(([b] * n for b, n in zip(bl, g["B"])), [])
    groups = [D.Group(n, p, bl[r - 1]) for n, p, r in zip(g["n"], g["p"], g["r"])]
    cost = [[int(100 * (k + 1) * (k + 2) / (1 + 0.8 * np.log2(n))) for k in range(4)] for n in g["n"]]
    res = D.dispatch(groups, cost, lens, [0] * len(lens), step, 1024, R=4)
    assert res.boundaries == bl
    assert res.r == [1, 2, 0, 4]
    assert res.d[:, 3].tolist() == [0, 0, 0, 4]
    assert res.d[2].sum() == 0
    assert res.d.sum(axis=0).tolist() == g["B"]
    # balanced dispatch dominates length-based dispatch
    res_len = D.dispatch(groups, cost, lens, [0] * len(lens), step, 1024, R=4, mode=1)
    assert res.t_hat <= res_len.t_hat


def _rand_instance(rng, G_max=3, R_max=3, B_max=6, p_max=2):
    G = int(rng.integers(1, G_max + 1))
    R = int(rng.integers(1, R_max + 1))
    Bj = rng.integers(0, B_max + 1, size=R)
    p = rng.integers(1, p_max + 1, size=G).tolist()
    r = sorted(rng.integers(1, R + 1, size=G).tolist())
    r[-1] = R
    c = [[int(x) for x in rng.integers(1, 20, size=R)] for _ in range(G)]
    return Bj, p, c, r


def test_eq3_milp_equals_bruteforce():
    """Exact optimum and canonical lexicographic d: HiGHS path == exhaustive path
    (S:292)."""
    rng = np.random.default_rng(13)
    for _ in range(40):
        Bj, p, c, r = _rand_instance(rng)
        d1, t1 = D.solve_bruteforce(Bj, p, c, r)
        d2, t2 = D.solve_milp(Bj, p, c, r)
        assert t1 == t2 and np.array_equal(d1, d2), (Bj, p, c, r)
        D.check_eq3(d1, Bj, p, r)


def test_eq3_single_group_and_cheaper_group():
    d, t = D.solve_bruteforce(np.array([3, 2]), [2], [[5, 7]], [2])
    assert d.tolist() == [[3, 2]] and t == 5 * 2 + 7 * 1
    d, t = D.solve_bruteforce(np.array([1]), [1, 1], [[9], [4]], [1, 1])
    assert d.tolist() == [[0], [1]] and t == 4


def test_dispatch_properties_random():
    """Conservation, per-replica ceil bound, memory limits, determinism on random
    multi-task batches."""
    rng = np.random.default_rng(14)
    groups = [D.Group(1, 2, 2048), D.Group(2, 1, 4096)]
    cost = [[(k + 1) * 3 for k in range(16)], [(k + 1) * 2 for k in range(16)]]
    for _ in range(5):
        n = int(rng.integers(5, 30))
        lens = rng.integers(1, 4096, size=n)
        tasks = rng.integers(0, 3, size=n)
        res = D.dispatch(groups, cost, lens, tasks, 256, 4096, R=4)
        res2 = D.dispatch(groups, cost, lens, tasks, 256, 4096, R=4)
        assert np.array_equal(res.seq_replica, res2.seq_replica)
        assert np.array_equal(res.pack_order, res2.pack_order)
        assert (res.seq_replica >= 0).all() and (res.pack_order >= 0).all()
        for rep in range(3):
            for j in range(len(res.boundaries)):
                i = 0 if rep < 2 else 1
                cnt = int(((res.seq_replica == rep) & (res.seq_bucket == j)).sum())
                assert cnt <= -(-int(res.d[i, j]) // groups[i].replicas)
        assert res.replica_cost.max() <= res.t_hat


def test_packed_chunking_respects_token_budget():
    """chunking=1 (packing): every chunk holds <= M_i real tokens; the C2-like
    16384-token pack on one replica with M = 16384 is exactly one chunk."""
    from workloads import synth
    wl = synth.config_c2()
    res = D.dispatch([D.Group(1, 1, 16384)], [[k + 1 for k in range(16)]], wl.seq_lens,
                     wl.seq_task, 256, 4096, R=16, chunking=1)
    assert set(res.seq_chunk.tolist()) == {0}
    rng = np.random.default_rng(3)
    lens = rng.integers(1, 2048, size=40)
    res = D.dispatch([D.Group(1, 2, 2048)], [[k + 1 for k in range(8)]], lens, lens % 3, 256,
                     2048, R=4, chunking=1)
    for rep in range(2):
        for c in set(res.seq_chunk[res.seq_replica == rep].tolist()):
            m = (res.seq_replica == rep) & (res.seq_chunk == c)
            assert lens[m].sum() <= 2048


# --------------------------------------------------------------------------- mode 1 pin
T3 = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table3_thruputs.json")))


def _table3_pp1_deployment():
    """The four PP = 1 configurations of Table tb:parallel_config_thruputs,
    one replica each, M = the longest length the table gives a throughput for, and the
    per-sequence cost = time of one sequence on one replica = s / (thruput * n) (tokens /
    (tokens per GPU per second * GPUs)), in integer units of 1e-6 s / 1e3."""
    rows = {tuple(c): T3["thruput"][k] for k, c in enumerate(T3["configs"])}
    lens = T3["seq_lens"]
    groups, cost = [], []
    for tp in (1, 2, 4, 8):
        th = rows[(tp, 1)]
        m = max(s for s, v in zip(lens, th) if v > 0)
        groups.append(D.Group(tp, 1, m))
        row = []
        for k in range(8):                      # grid 2048 .. 16384
            s = 2048 * (k + 1)
            v = dict(zip(lens, th)).get(s, 0) or min(x for x in th if x > 0)
            row.append(int(round(1e6 * s / (v * tp))))
        cost.append(row)
    return groups, cost


def test_length_based_mode_sends_each_bucket_to_the_most_efficient_config():
    """Fig. 4(c): length-based dispatch sends every bucket to 'the most
    suitable replica(s)' so that 'from the perspective of each sequence, it can be processed
    by the most efficient configuration' -- the highest tokens per GPU per second of Table
    tb:parallel_config_thruputs.  Hand-read from the table: 2K -> TP1 (5.11 > 4.30 > 3.63 >
    2.79), 4K -> TP2 (4.12 > 3.50 > 2.71), 8K -> TP4 (3.25 > 2.56), 16K -> TP8 (2.33, the only
    one).  A rule that minimised the per-replica time c_ij alone (ignoring the n_i GPUs it
    occupies) would send every bucket to TP8 instead."""
    groups, cost = _table3_pp1_deployment()
    lens = [2048] * 5 + [4096] * 3 + [8192] * 2 + [16384]
    res = D.dispatch(groups, cost, lens, [0] * len(lens), 2048, 16384, 4, mode=1)
    assert res.boundaries == [2048, 4096, 8192, 16384]
    assert res.d.tolist() == [[5, 0, 0, 0], [0, 3, 0, 0], [0, 0, 2, 0], [0, 0, 0, 1]]
    # the per-replica-time rule differs on this instance (the pin has teeth)
    by_c = [min(range(4), key=lambda i: (cost[i][b // 2048 - 1] if b <= groups[i].max_tokens else 1e18, i))
            for b in res.boundaries]
    assert by_c == [3, 3, 3, 3]


def test_length_based_mode_cpp_matches_hand_reading():
    from paper_2509_01193_b200 import _lib
    groups, cost = _table3_pp1_deployment()
    lens = [2048] * 5 + [4096] * 3 + [8192] * 2 + [16384]
    got = _lib.lobra_dispatch([g.tp for g in groups], [1] * 4, [g.max_tokens for g in groups], cost, lens,
                              [0] * len(lens), 2048, 16384, 4, mode=1)
    assert got["d"].tolist() == [[5, 0, 0, 0], [0, 3, 0, 0], [0, 0, 2, 0], [0, 0, 0, 1]]


# --------------------------------------------------------------------------- steps 9-10 pins
def test_chunks_and_packing_order_hand_worked():
    """Steps 9-10 of the oracle by hand, one replica (M = 1024, grid 256, R = 2).
    Lengths (index: len, task): 0:200 t2, 1:900 t0, 2:250 t1, 3:100 t0, 4:700 t1, 5:60 t2.
    Grid values 256 (0, 2, 3, 5) and 1024 (1, 4) -> buckets [256, 1024].
    chunking = 0 (App. D, b_j = floor(M / s_j)): bucket 1024 -> b = 1 -> chunks {1}, {4};
      bucket 256 -> b = 4 -> chunk {0, 2, 3, 5}; descending cost c_j * count with cost 1 per
      256 tokens: {0,2,3,5} costs 4, {1} and {4} cost 4 each -> ties by bucket index: the
      256-bucket chunk first, then {1}, {4}.  Inside a chunk: (task, index) -> 3, 2, 0, 5.
    chunking = 1 (packed next-fit over (bucket desc, index asc) = 1, 4, 0, 2, 3, 5 with at
      most M real tokens): {1} (900; +700 overflows), {4, 0} (900; +250 overflows),
      {2, 3, 5} (410).  Chunks in creation order; packing inside by (task, index): {1};
      {4 (t1), 0 (t2)}; {3 (t0), 2 (t1), 5 (t2)}."""
    groups = [D.Group(1, 1, 1024)]
    lens = [200, 900, 250, 100, 700, 60]
    tasks = [2, 0, 1, 0, 1, 2]
    cost = [[1, 2, 3, 4]]
    r0 = D.dispatch(groups, cost, lens, tasks, 256, 1024, 2, chunking=0)
    assert r0.boundaries == [256, 1024]
    assert r0.seq_chunk.tolist() == [0, 1, 0, 0, 2, 0]
    assert r0.pack_order.tolist() == [2, 0, 1, 0, 0, 3]
    r1 = D.dispatch(groups, cost, lens, tasks, 256, 1024, 2, chunking=1)
    assert r1.seq_chunk.tolist() == [1, 0, 2, 2, 1, 2]
    assert r1.pack_order.tolist() == [1, 0, 1, 0, 0, 2]


# --------------------------------------------------------------------------- steps 9-10 pin
def test_micro_batches_and_packing_order_hand_worked():
    """Steps 9-10 (padded micro-batches of App. D P:1494-1496 in descending cost; packed
    next-fit chunks, reading Q6b; task-grouped order inside a chunk, reading Q6) against a
    hand-worked instance (tests/golden/dispatch_pack_example.json, derivation inside)."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "dispatch_pack_example.json")))
    groups = [D.Group(*g["group"])]
    for chunking, key in ((0, "padded"), (1, "packed")):
        res = D.dispatch(groups, [g["cost"]], np.array(g["seq_lens"]), np.array(g["seq_task"]), g["grid_step"],
                         g["grid_max"], g["R"], mode=0, chunking=chunking)
        assert list(res.boundaries) == g["boundaries"]
        assert [int(x) for x in np.asarray(res.d).ravel()] == g["d"]
        assert int(res.t_hat) == g["t_hat"]
        assert res.seq_chunk.tolist() == g[key]["seq_chunk"], key
        assert res.pack_order.tolist() == g[key]["pack_order"], key
