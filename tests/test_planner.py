"""Stage-1 deployment planning: the oracle pinned to the paper's §3
worked instance (with the paper's Table 3 throughputs), the C++ planner == the oracle,
pruning safety, Theorem-1 soundness on proportional cost laws.  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import planner as PL
from workloads import synth

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "planner_design_anatomy.json")))


def _fixture_cost():
    """[S][U] integer costs on the 2048 grid (U = 8) from Table 3 throughputs."""
    U = 8
    thr = {int(k): {int(s): v for s, v in d.items()} for k, d in G["throughput_k_tokens_per_gpu_s"].items()}
    cost = []
    for n in G["tp"]:
        row = []
        for k in range(U):
            s = (k + 1) * 2048
            ok = [L for L in sorted(thr[n]) if L >= s]
            v = s / (thr[n][ok[0]] * n) if ok else 0.0       # padded to the config's next row
            row.append(int(round(v / G["cost_unit_ms"])))
        cost.append(row)
    M = [max(thr[n]) for n in G["tp"]]
    lens = sum(([L] * B for L, B in zip(G["bucket_lengths"], G["demands"])), [])
    return M, cost, lens


def test_oracle_reproduces_paper_design_anatomy():
    """'the numbers of deployed replicas with the configurations are {4,2,0,1}'."""
    M, cost, lens = _fixture_cost()
    joint = PL.solve_joint(G["tp"], M, cost, G["n_gpus"], (G["bucket_lengths"], G["demands"]), 2048)
    assert joint[3] == G["expected_replicas"]
    res = PL.plan_deployment(G["tp"], M, cost, G["n_gpus"], lens, 0, 2048, 16384, 4, threshold=-1)
    assert res["replicas"] == G["expected_replicas"]
    assert res["t_hat"] == joint[0]


def test_cpp_planner_design_anatomy():
    from paper_2509_01193_b200 import _lib
    M, cost, lens = _fixture_cost()
    for thr in (-1.0, 0.15):
        got = _lib.lobra_plan_deployment(G["tp"], M, cost, G["n_gpus"], lens, 0, 2048, 16384, 4,
                                         threshold=thr)
        assert got["replicas"].tolist() == G["expected_replicas"]
        assert got["demands"].tolist() == G["demands"]


def _rand_problem(seed):
    rng = np.random.default_rng(seed)
    tps = [1, 2, 4]
    M = [2048, 4096, 8192]
    thr = {1: 5.0, 2: 4.3, 4: 3.4}
    # proportional law with a mild length penalty; integer units
    cost = [[max(1, int(round((k + 1) * 256 / (thr[n] * n) * (1 + 0.02 * k) / 8))) for k in range(32)]
            for n in tps]
    tasks = synth.c3_tasks()
    wl = synth.sample_batch(tasks, seed=seed, l_max=8192, per_task=[int(x) for x in rng.integers(2, 6, size=16)])
    return tps, M, cost, wl


@pytest.mark.parametrize("seed", range(5))
def test_cpp_planner_equals_oracle(seed):
    from paper_2509_01193_b200 import _lib
    tps, M, cost, wl = _rand_problem(seed)
    N = int(np.random.default_rng(seed).integers(3, 9))
    for thr in (-1.0, 0.15):
        ref = PL.plan_deployment(tps, M, cost, N, wl.seq_lens, 40, 256, 8192, 4, threshold=thr)
        got = _lib.lobra_plan_deployment(tps, M, cost, N, wl.seq_lens, 40, 256, 8192, 4, threshold=thr)
        assert got["replicas"].tolist() == ref["replicas"], (thr, got, ref)
        assert got["t_hat"] == ref["t_hat"]
        assert got["plans_total"] == ref["plans_total"] and got["plans_solved"] == ref["plans_solved"]
        assert got["demands"].tolist() == ref["demands"].tolist()


def test_pruning_safe_on_paper_fixture_and_theorem1():
    """App. A: the 15% lower-bound filter keeps the unfiltered plan on the paper's fixture
    (it is a heuristic in general, so only checked there); Theorem 1: the exact
    balanced optimum t_hat of every plan is >= the length-based bound (proportional law)."""
    M, cost, lens = _fixture_cost()
    a = PL.plan_deployment(G["tp"], M, cost, G["n_gpus"], lens, 0, 2048, 16384, 4, threshold=-1)
    b = PL.plan_deployment(G["tp"], M, cost, G["n_gpus"], lens, 0, 2048, 16384, 4, threshold=0.15)
    assert a["replicas"] == b["replicas"] and a["t_hat"] == b["t_hat"]
    for seed in range(3):
        tps, Ms, costs, wl = _rand_problem(10 + seed)
        bounds, Bj = PL._buckets(wl.seq_lens, 256, 8192, 4, 40)
        r, c = PL._tables(tps, Ms, costs, bounds, 256)
        for p in PL._plans(tps, [True] * 3, r, Bj, 8):
            t = PL._solve_plan(p, tps, r, c, Bj)
            assert t >= PL.lower_bound(p, tps, r, c, Bj) - 1e-9


def test_single_candidate():
    from paper_2509_01193_b200 import _lib
    got = _lib.lobra_plan_deployment([2], [4096], [[k + 1 for k in range(16)]], 7, [100, 900, 3000],
                                     0, 256, 4096, 4)
    assert got["replicas"].tolist() == [3] and got["gpus_used"] == 6


# ---------------------------------------------------------------- configuration proposal
T3 = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table3_thruputs.json")))


def _t3():
    tp = [c[0] for c in T3["configs"]]
    pp = [c[1] for c in T3["configs"]]
    return tp, pp, T3["seq_lens"], T3["thruput"], T3["gpu_counts"]


def test_oracle_proposal_selects_the_bold_configs_of_table3():
    """App. A: the proposal on Table tb:parallel_config_thruputs keeps exactly the bolded
    configurations, each winning the cell the paper bolds (P:918 5.11, P:960 2.33,
    P:971 3.79, ...)."""
    tp, pp, sl, th, gc = _t3()
    win, keep = PL.propose_from_table(tp, pp, sl, th, gc)
    kept = sorted(T3["configs"][c] for c in range(len(tp)) if keep[c])
    assert kept == sorted(T3["expected_bold"])
    for cell in T3["expected_cells"]:
        c = win[gc.index(cell["num_gpus"])][sl.index(cell["seq_len"])]
        assert T3["configs"][c] == cell["config"]
        assert th[c][sl.index(cell["seq_len"])] == cell["thruput"]
    # without replication the (2 GPUs, 2K) group would pick <TP=1,PP=2> (4.88, not bold)
    assert T3["configs"][win[gc.index(2)][sl.index(2048)]] == [1, 1]
    # no configuration runs 4K on one GPU
    assert win[gc.index(1)][sl.index(4096)] == -1


def test_observation1_holds_on_table3():
    """the paper's table is consistent with the partial order (Observation 1)."""
    assert PL.check_partial_order(*_t3()) == []
    # a planted inversion is reported
    tp, pp, sl, th, gc = _t3()
    th = [list(r) for r in th]
    th[8][0] = 3.0      # <TP=2,PP=4> now slower than <TP=4,PP=1> at 2K but faster at 8K
    v = PL.check_partial_order(tp, pp, sl, th, gc)
    assert (8, 8, 3, 8192, 2048) in v


def test_proposal_single_config_and_ties():
    win, keep = PL.propose_from_table([2], [1], [1024], [[1.0]], [2, 4])
    assert keep == [1] and win == [[0], [0]]
    # equal throughput: fewer GPUs per replica, then smaller TP, then smaller PP
    win, keep = PL.propose_from_table([2, 1, 1], [1, 2, 1], [512], [[3.0], [3.0], [3.0]], [2])
    assert win == [[2]]
    win, keep = PL.propose_from_table([2, 1], [1, 2], [512], [[3.0], [3.0]], [2])
    assert win == [[1]]


def test_cpp_proposal_equals_oracle():
    from paper_2509_01193_b200 import _lib
    tp, pp, sl, th, gc = _t3()
    win, keep = _lib.lobra_propose_configs(tp, pp, sl, th, gc)
    ow, ok = PL.propose_from_table(tp, pp, sl, th, gc)
    assert win.tolist() == ow and keep.tolist() == ok
    rng = np.random.default_rng(7)
    for _ in range(300):
        C = int(rng.integers(1, 9))
        L = int(rng.integers(1, 5))
        tp = rng.choice([1, 2, 4, 8], C).tolist()
        pp = rng.choice([1, 2, 4], C).tolist()
        th = np.round(rng.uniform(-1, 5, (C, L)), 1)     # coarse values force ties; <= 0 = OOM
        gc = sorted(set(rng.choice([1, 2, 4, 8, 16, 32], int(rng.integers(1, 4))).tolist()))
        sl = [256 * (i + 1) for i in range(L)]
        win, keep = _lib.lobra_propose_configs(tp, pp, sl, th, gc)
        ow, ok = PL.propose_from_table(tp, pp, sl, th.tolist(), gc)
        assert win.tolist() == ow and keep.tolist() == ok


def test_cpp_proposal_errors():
    from paper_2509_01193_b200 import _lib
    with pytest.raises(_lib.LobraError):
        _lib.lobra_propose_configs([0], [1], [512], [[1.0]], [1])
    with pytest.raises(_lib.LobraError):
        _lib.lobra_propose_configs([1], [1], [512], [[1.0]], [0])
