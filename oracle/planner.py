"""Integer oracle of LobRA's stage-1 deployment planning -- TEST INFRASTRUCTURE ONLY.

Follows §4.2 (Eq. 2) and App. A step by step (PP = 1):
 1. dynamic bucketing of a length sample, 2. demands B_j = ceil(B f_j)
 (reading Q22; B = 0 -> the sample's counts), 3. configuration proposal (App. A
 Observation 1: drop a candidate dominated by another with the same GPU count),
 4. maximal covering plans sum p_i n_i <= N (App. A "integer partition"), 5. Theorem-1
 lower bound sum_i N_i t_i / sum_i N_i with length-based dispatch times t_i, filter at
 (1 + threshold) x the minimum bound, 6. exact Eq. 3 per kept plan (oracle.dispatch), best
 by (t_hat, GPUs, replicas, lexicographic p).  ``solve_joint`` = Eq. 1 over ALL plans
 (not only maximal, no filtering) for pinning.
"""
from __future__ import annotations

import itertools

import numpy as np

from . import dispatch as D


def _buckets(lens, grid_step, grid_max, R, batch_size):
    counts = D.histogram(lens, grid_step, grid_max)
    bounds, _ = D.dynamic_buckets(counts, grid_step, R)
    cnt = []
    prev = 0
    for s in bounds:
        k = s // grid_step
        cnt.append(int(counts[prev:k].sum()))
        prev = k
    n = len(lens)
    Bj = [-(-batch_size * c // n) if batch_size > 0 else c for c in cnt]
    return bounds, np.array(Bj, np.int64)


def _tables(tp, max_tokens, cost, bounds, grid_step):
    S = len(tp)
    r = [sum(1 for s in bounds if s <= max_tokens[i]) for i in range(S)]
    c = [[int(cost[i][s // grid_step - 1]) for s in bounds] for i in range(S)]
    return r, c


def propose(tp, r, c):
    """App. A Observation 1: keep[i] = False if another candidate with the same GPU count
    supports >= buckets at <= cost (strictly better somewhere, or equal and earlier)."""
    S = len(tp)
    keep = [True] * S
    for a in range(S):
        for b in range(S):
            if a == b or not keep[a] or not keep[b] or tp[a] != tp[b] or r[b] < r[a]:
                continue
            if all(c[b][j] <= c[a][j] for j in range(r[a])):
                strict = r[b] > r[a] or any(c[b][j] < c[a][j] for j in range(r[a]))
                if strict or b < a:
                    keep[a] = False
    return keep


def _plans(tp, keep, r, Bj, N, maximal=True):
    S = len(tp)
    last = max([j for j in range(len(Bj)) if Bj[j] > 0], default=-1)
    ranges = [range(N // tp[i] + 1) if keep[i] else range(1) for i in range(S)]
    min_n = min(tp[i] for i in range(S) if keep[i])
    out = []
    for p in itertools.product(*ranges):
        used = sum(p[i] * tp[i] for i in range(S))
        if used > N or used == 0:
            continue
        if maximal and N - used >= min_n:
            continue
        cover = max([r[i] for i in range(S) if p[i] > 0], default=0)
        if cover - 1 < last:
            continue
        out.append(list(p))
    return out


def _solve_plan(p, tp, r, c, Bj):
    live = [i for i in range(len(p)) if p[i] > 0]
    d, t = D.solve_eq3(Bj, [p[i] for i in live], [c[i] for i in live], [r[i] for i in live],
                       bruteforce_cap=20000)
    return t


def _key(t, p, tp):
    return (t, sum(a * b for a, b in zip(p, tp)), sum(p), list(p))


def lower_bound(p, tp, r, c, Bj):
    """Theorem 1 (App. A): sum_i N_i t_i / sum_i N_i with length-based dispatch (each
    bucket to the supporting deployed group with the smallest c_ij n_i)."""
    live = [i for i in range(len(p)) if p[i] > 0]
    t = {i: 0 for i in live}
    for j in range(len(Bj)):
        if Bj[j] == 0:
            continue
        best = min((c[i][j] * tp[i], i) for i in live if j < r[i])[1]
        t[best] += c[best][j] * (-(-int(Bj[j]) // p[best]))
    num = sum(p[i] * tp[i] * t[i] for i in live)
    den = sum(p[i] * tp[i] for i in live)
    return num / den


def plan_deployment(tp, max_tokens, cost, N, lens, batch_size=0, grid_step=256, grid_max=16384,
                    R=16, threshold=0.15):
    bounds, Bj = _buckets(lens, grid_step, grid_max, R, batch_size)
    r, c = _tables(tp, max_tokens, cost, bounds, grid_step)
    keep = propose(tp, r, c)
    plans = _plans(tp, keep, r, Bj, N, maximal=True)
    if not plans:
        raise D.DispatchError(2, "no plan covers the longest bucket")
    lbs = [lower_bound(p, tp, r, c, Bj) for p in plans]
    m = min(lbs)
    best, solved = None, 0
    for p, lb in zip(plans, lbs):
        if threshold >= 0 and lb > (1 + threshold) * m + 1e-9:
            continue
        solved += 1
        k = _key(_solve_plan(p, tp, r, c, Bj), p, tp)
        if best is None or k < best:
            best = k
    return {"replicas": best[3], "t_hat": best[0], "boundaries": bounds, "demands": Bj,
            "plans_total": len(plans), "plans_solved": solved, "gpus_used": best[1]}


def solve_joint(tp, max_tokens, cost, N, Bj_bounds, grid_step):
    """Eq. 1 with concrete demands over ALL feasible plans (no proposal, no filtering)."""
    bounds, Bj = Bj_bounds
    r, c = _tables(tp, max_tokens, cost, bounds, grid_step)
    best = None
    for p in _plans(tp, [True] * len(tp), r, np.asarray(Bj), N, maximal=False):
        k = _key(_solve_plan(p, tp, r, c, np.asarray(Bj)), p, tp)
        if best is None or k < best:
            best = k
    return best


# ------------------------------------------------------------------------------------------
# Configuration proposal from a profiled throughput table (App. A; Table
# tb:parallel_config_thruputs).  Reading Q26: a configuration with
# n_c = tp * pp GPUs per replica competes in every (num_gpus = g, seq_len) group with
# n_c <= g and n_c | g, as g / n_c replicas at its own per-GPU throughput (the table's "-":
# "the throughput remains the same after model replication"); the winner of a group is the
# maximum throughput ("SELECT config, MAX(thruput) ... GROUP BY num_gpus, seq_len"), ties to
# fewer GPUs per replica, then smaller TP, then smaller PP, then table order.
# ------------------------------------------------------------------------------------------
def propose_from_table(tp, pp, seq_lens, thruput, gpu_counts):
    """Returns (winner[g][l] config index or -1, keep[c] 0/1).  thruput[c][l] <= 0 means the
    configuration cannot run that length (the table's out-of-memory mark)."""
    C = len(tp)
    winner = []
    for g in gpu_counts:
        row = []
        for li in range(len(seq_lens)):
            best = -1
            for c in range(C):
                n = tp[c] * pp[c]
                if n > g or g % n != 0 or not thruput[c][li] > 0:
                    continue
                if best < 0:
                    best = c
                    continue
                kc = (-thruput[c][li], n, tp[c], pp[c], c)
                kb = (-thruput[best][li], tp[best] * pp[best], tp[best], pp[best], best)
                if kc < kb:
                    best = c
            row.append(best)
        winner.append(row)
    keep = [0] * C
    for row in winner:
        for c in row:
            if c >= 0:
                keep[c] = 1
    return winner, keep


def check_partial_order(tp, pp, seq_lens, thruput, gpu_counts):
    """Observation 1 on the replication-inclusive table: for every GPU count g,
    configurations alpha, beta runnable on g GPUs and lengths s < s0 where both run at both:
    alpha faster at s0 must be faster at s.  Returns the violations (g, alpha, beta, s0, s)."""
    out = []
    C = len(tp)
    L = len(seq_lens)
    for g in gpu_counts:
        cfg = [c for c in range(C) if tp[c] * pp[c] <= g and g % (tp[c] * pp[c]) == 0]
        for a in cfg:
            for b in cfg:
                if a == b:
                    continue
                for l0 in range(L):
                    if not (thruput[a][l0] > 0 and thruput[b][l0] > 0):
                        continue
                    if not thruput[a][l0] > thruput[b][l0]:
                        continue
                    for l in range(l0):
                        if thruput[a][l] > 0 and thruput[b][l] > 0 and not thruput[a][l] > thruput[b][l]:
                            out.append((g, a, b, seq_lens[l0], seq_lens[l]))
    return out
