"""C++ lobra_dispatch vs the integer oracle: bit-exact on every output (CPU only)."""
import json
import os

import numpy as np
import pytest

from oracle import dispatch as D
from workloads import synth

pytestmark = []


def _run_both(groups, cost, lens, tasks, step, gmax, R, mode=0, cap=200000, chunking=0):
    from paper_2509_01193_b200 import _lib
    ref = D.dispatch(groups, cost, lens, tasks, step, gmax, R, mode=mode, bruteforce_cap=cap,
                     chunking=chunking)
    got = _lib.lobra_dispatch([g.tp for g in groups], [g.replicas for g in groups],
                              [g.max_tokens for g in groups], cost, lens, tasks, step, gmax, R, mode,
                              chunking=chunking)
    assert got["status"] == 0
    assert got["boundaries"].tolist() == ref.boundaries
    assert np.array_equal(got["d"], ref.d), (got["d"], ref.d)
    assert got["t_hat"] == ref.t_hat
    assert np.array_equal(got["seq_bucket"], ref.seq_bucket)
    assert np.array_equal(got["seq_replica"], ref.seq_replica)
    assert np.array_equal(got["seq_chunk"], ref.seq_chunk)
    assert np.array_equal(got["pack_order"], ref.pack_order)
    assert np.array_equal(got["replica_cost"][:len(ref.replica_cost)], ref.replica_cost)
    return got, ref


def _cost_table(groups, U, step, rng=None, a1=1.0, a2=0.0, unit=1.0):
    """Integer per-sequence costs ~ (a1 s + a2 s^2) / tp-efficiency (App. D shape)."""
    out = []
    for g in groups:
        eff = g.tp * (0.85 ** np.log2(g.tp))
        row = []
        for k in range(U):
            s = (k + 1) * step
            row.append(max(1, int(round((a1 * s + a2 * s * s) / eff / unit))))
        out.append(row)
    return out


def test_spec_examples_cpp():
    _run_both([D.Group(1, 1, 8)], [[4, 8]], [4] * 5, [0] * 5, 4, 8, 1)
    _run_both([D.Group(1, 2, 8)], [[4, 8]], [4] * 5, [0] * 5, 4, 8, 1)


def test_design_anatomy_cpp():
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                    "dispatch_spec_examples.json")))["design_anatomy"]
    bl = [256, 512, 768, 1024]
    lens = sum(([b] * n for b, n in zip(bl, g["B"])), [])
    groups = [D.Group(n, p, bl[r - 1]) for n, p, r in zip(g["n"], g["p"], g["r"])]
    cost = [[int(100 * (k + 1) * (k + 2) / (1 + 0.8 * np.log2(n))) for k in range(4)] for n in g["n"]]
    got, ref = _run_both(groups, cost, lens, [0] * len(lens), 256, 1024, 4)
    _run_both(groups, cost, lens, [0] * len(lens), 256, 1024, 4, mode=1)


@pytest.mark.parametrize("seed", range(12))
def test_random_small_bruteforce(seed):
    rng = np.random.default_rng(100 + seed)
    G = int(rng.integers(1, 4))
    groups = []
    for i in range(G):
        groups.append(D.Group(2 ** i, int(rng.integers(1, 3)), 256 * (i + 1) * 2))
    n = int(rng.integers(1, 9))
    gmax = groups[-1].max_tokens
    lens = rng.integers(1, gmax + 1, size=n)
    tasks = rng.integers(0, 3, size=n)
    U = gmax // 256
    cost = [[int(x) for x in rng.integers(1, 30, size=U)] for _ in groups]
    _run_both(groups, cost, lens, tasks, 256, gmax, int(rng.integers(1, 5)))


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("chunking", [0, 1])
def test_two_groups_milp_scale(seed, chunking):
    """G=2 (TP1 x p1 + TP2 x p2) on skewed multi-task batches: C++ exact DP == oracle
    HiGHS + lexicographic canonicalisation."""
    rng = np.random.default_rng(200 + seed)
    groups = [D.Group(1, int(rng.integers(1, 5)), 2048), D.Group(2, int(rng.integers(1, 3)), 4096)]
    tasks = synth.c2_tasks()
    wl = synth.sample_batch(tasks, seed=300 + seed, l_max=4096, per_task=[12, 8, 8, 4])
    cost = _cost_table(groups, 4096 // 256, 256, a1=1.0, a2=1.0 / 8192, unit=64)
    _run_both(groups, cost, wl.seq_lens, wl.seq_task, 256, 4096, 6, cap=2000, chunking=chunking)


def test_three_groups_cpp():
    rng = np.random.default_rng(7)
    groups = [D.Group(1, 2, 1024), D.Group(2, 1, 2048), D.Group(4, 1, 4096)]
    lens = rng.integers(1, 4096, size=14)
    tasks = rng.integers(0, 4, size=14)
    cost = _cost_table(groups, 16, 256, a1=1.0, unit=128)
    _run_both(groups, cost, lens, tasks, 256, 4096, 4, cap=2000)


def test_errors_cpp():
    from paper_2509_01193_b200 import _lib
    with pytest.raises(_lib.LobraError) as e:
        _lib.lobra_dispatch([1], [1], [512], [[1, 2]], [600], [0], 256, 512, 2)
    assert e.value.status == _lib.LOBRA_ERR_INFEASIBLE
    with pytest.raises(_lib.LobraError) as e:   # sequence longer than every replica limit
        _lib.lobra_dispatch([1], [1], [256], [[1, 2]], [300], [0], 256, 512, 2)
    assert e.value.status == _lib.LOBRA_ERR_INFEASIBLE
    with pytest.raises(_lib.LobraError) as e:   # groups out of (tp, M) order
        _lib.lobra_dispatch([2, 1], [1, 1], [512, 512], [[1, 2], [1, 2]], [100], [0], 256, 512, 2)
    assert e.value.status == _lib.LOBRA_ERR_INPUT


def test_c5_scale_runs_fast():
    """C5-like step: 4xTP1 (M=8192) + 2xTP2 (M=16384), 16 tasks' batch (~1950 seqs),
    R=16 -- exact, canonical, and well under a second (P:586 'fully overlapped')."""
    import time
    from paper_2509_01193_b200 import _lib
    tasks = synth.c3_tasks()
    wl = synth.sample_batch(tasks, seed=100, l_max=16384, per_task=[t.batch_size for t in tasks[:12]] + [64] * 4)
    groups = [D.Group(1, 4, 8192), D.Group(2, 2, 16384)]
    cost = _cost_table(groups, 64, 256, a1=1.0, a2=1.0 / 16384, unit=32)
    t0 = time.time()
    got = _lib.lobra_dispatch([1, 2], [4, 2], [8192, 16384], cost, wl.seq_lens, wl.seq_task, 256, 16384, 16)
    dt = time.time() - t0
    assert got["status"] == 0 and dt < 5.0
    assert got["d"].sum() == len(wl.seq_lens)
    # sequences longer than 8192 never reach a TP1 replica
    long = wl.seq_lens > 8192
    assert (got["seq_replica"][long] >= 4).all()


# --------------------------------------------------------------------------- C5 scale, G = 2..4
_C5 = os.path.join(os.path.dirname(__file__), "golden", "dispatch_c5.json")
C5 = json.load(open(_C5)) if os.path.exists(_C5) else {"cases": []}


def _c5_cost(groups, unit):
    out = []
    for g in groups:
        eff = g.tp * (0.85 ** np.log2(g.tp))
        out.append([max(1, int(round(((k + 1) * 256 + ((k + 1) * 256) ** 2 / 16384) / eff / unit)))
                    for k in range(64)])
    return out


def _digest(*arrays):
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("case", C5["cases"], ids=lambda c: f"{c['name']}-s{c['seed']}")
def test_c5_scale_exact_vs_oracle_fixture(case):
    """C5-scale steps (B ~ 1952 sequences of C3's 16 tasks, R = 16) on 2-4 deployed groups
    (TP1/TP2/TP4/TP8): the C++ Eq. 3 solver returns exactly the oracle's optimum and
    canonical (lexicographically smallest) d, and the same per-sequence outputs
    (tests/golden/dispatch_c5.json, written by tools/gen_dispatch_golden.py from the
    oracle alone)."""
    import time
    from paper_2509_01193_b200 import _lib
    groups = [D.Group(*g) for g in case["deployment"]]
    cost = _c5_cost(groups, C5["cost_unit"])
    tasks = synth.c3_tasks()
    wl = synth.sample_batch(tasks, seed=case["seed"], l_max=16384,
                            per_task=[t.batch_size for t in tasks[:12]] + [64] * 4)
    assert len(wl.seq_lens) == case["num_seqs"]
    t0 = time.perf_counter()
    got = _lib.lobra_dispatch([g.tp for g in groups], [g.replicas for g in groups],
                              [g.max_tokens for g in groups], cost, wl.seq_lens, wl.seq_task,
                              C5["grid_step"], C5["grid_max"], C5["R"], 0, chunking=C5["chunking"])
    dt = time.perf_counter() - t0
    assert got["status"] == 0
    assert got["boundaries"].tolist() == case["boundaries"]
    assert got["t_hat"] == case["t_hat"]
    assert got["d"].tolist() == case["d"]
    assert _digest(got["seq_bucket"], got["seq_replica"], got["seq_chunk"], got["pack_order"],
                   got["replica_cost"]) == case["sha256"]
    assert dt < 10.0, dt   # measured solve times: profiles/r2_dispatch_solve_times.md


@pytest.mark.parametrize("threads", ["1", "3"])
def test_c5_scale_thread_count_invariant(threads, monkeypatch):
    """The >= 3-group solver explores subtrees on a thread pool (LOBRA_DISPATCH_THREADS):
    the answer, including every per-sequence output, is the fixture's for any thread count."""
    from paper_2509_01193_b200 import _lib
    cases = [c for c in C5["cases"] if c["name"] in ("G3", "G4")][:2]
    if not cases:
        pytest.skip("no C5 fixture")
    monkeypatch.setenv("LOBRA_DISPATCH_THREADS", threads)
    for case in cases:
        groups = [D.Group(*g) for g in case["deployment"]]
        cost = _c5_cost(groups, C5["cost_unit"])
        tasks = synth.c3_tasks()
        wl = synth.sample_batch(tasks, seed=case["seed"], l_max=16384,
                                per_task=[t.batch_size for t in tasks[:12]] + [64] * 4)
        got = _lib.lobra_dispatch([g.tp for g in groups], [g.replicas for g in groups],
                                  [g.max_tokens for g in groups], cost, wl.seq_lens, wl.seq_task,
                                  C5["grid_step"], C5["grid_max"], C5["R"], 0, chunking=C5["chunking"])
        assert got["d"].tolist() == case["d"]
        assert _digest(got["seq_bucket"], got["seq_replica"], got["seq_chunk"], got["pack_order"],
                       got["replica_cost"]) == case["sha256"]


def test_c5_scale_live_oracle_g3():
    """One C5-scale 3-group step against the live oracle (not the fixture)."""
    tasks = synth.c3_tasks()
    wl = synth.sample_batch(tasks, seed=107, l_max=16384,
                            per_task=[t.batch_size for t in tasks[:12]] + [64] * 4)
    groups = [D.Group(1, 2, 8192), D.Group(2, 1, 16384), D.Group(4, 1, 16384)]
    _run_both(groups, _c5_cost(groups, 32), wl.seq_lens, wl.seq_task, 256, 16384, 16, chunking=1)


def test_budget_exhaustion_is_loud():
    """A node budget too small for Eq. 3 raises (LOBRA_ERR_BUDGET) instead of silently
    returning the length-based d; allow_budget=True returns it with the status."""
    from paper_2509_01193_b200 import _lib
    tasks = synth.c3_tasks()
    wl = synth.sample_batch(tasks, seed=100, l_max=16384,
                            per_task=[t.batch_size for t in tasks[:12]] + [64] * 4)
    groups = [D.Group(1, 2, 8192), D.Group(2, 1, 16384), D.Group(4, 1, 16384)]
    args = ([1, 2, 4], [2, 1, 1], [8192, 16384, 16384], _c5_cost(groups, 32), wl.seq_lens, wl.seq_task,
            256, 16384, 16, 0)
    with pytest.raises(_lib.LobraError) as e:
        _lib.lobra_dispatch(*args, node_cap=5)
    assert e.value.status == _lib.LOBRA_ERR_BUDGET
    got = _lib.lobra_dispatch(*args, node_cap=5, allow_budget=True)
    assert got["status"] == _lib.LOBRA_ERR_BUDGET


def test_uniform_mode_cpp():
    rng = np.random.default_rng(9)
    lens = rng.integers(1, 4096, size=37)
    tasks = rng.integers(0, 4, size=37)
    groups = [D.Group(2, 4, 4096)]
    cost = _cost_table(groups, 16, 256, a1=1.0, unit=64)
    got, ref = _run_both(groups, cost, lens, tasks, 256, 4096, 8, mode=2, chunking=1)
    assert np.bincount(got["seq_replica"]).tolist() == [10, 9, 9, 9]
    from paper_2509_01193_b200 import _lib
    with pytest.raises(_lib.LobraError):
        _lib.lobra_dispatch([1, 2], [2, 1], [2048, 4096], _cost_table([D.Group(1, 2, 2048), D.Group(2, 1, 4096)], 16, 256),
                            lens, tasks, 256, 4096, 8, 2)


def test_micro_batches_and_packing_order_hand_worked_cpp():
    """The C++ steps 9-10 on the hand-worked instance (tests/golden/dispatch_pack_example.json)."""
    from paper_2509_01193_b200 import _lib
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "dispatch_pack_example.json")))
    tp, p, M = g["group"]
    for chunking, key in ((0, "padded"), (1, "packed")):
        got = _lib.lobra_dispatch([tp], [p], [M], [g["cost"]], g["seq_lens"], g["seq_task"], g["grid_step"],
                                  g["grid_max"], g["R"], 0, chunking=chunking)
        assert got["boundaries"].tolist() == g["boundaries"]
        assert got["d"].ravel().tolist() == g["d"] and got["t_hat"] == g["t_hat"]
        assert got["seq_chunk"].tolist() == g[key]["seq_chunk"], key
        assert got["pack_order"].tolist() == g[key]["pack_order"], key
