"""Replica time cost model of App. D -- TEST INFRASTRUCTURE ONLY.

Follows PAPER.md App. D step by step, in the paper's notation:

* bucket j holds d_j sequences of (padded) length s_j; a configuration S with maximum
  supportable sequence length M (tokens per micro-batch, the OOM boundary) runs full chunks
  of b_j = floor(M / s_j) sequences: d_j = m_j * b_j + r_j  (Eq. appendix_cost_model_w/o_pp,
  P:1491-1497; the remainder r_j is renamed ``rem`` as in reading Q20);
* without pipeline parallel:  T = sum_j ( m_j * t(b_j, s_j) + t(r_j, s_j) );
* 1F1B with p stages, variable lengths (Eq. appendix_cost_model_pp_varlen):
  T = sum_j ( m_j * t(b_j, s_j) + t(r_j, s_j) )  +  (p - 1) * max_j { t(b_j, s_j), t(r_j, s_j) };
* fixed length (Eq. appendix_cost_model_pp_fixed_len):
  T(b, s, m) = m * t(b / m, s) + (p - 1) * t(b / m, s).

Reading (Q29): the max of the bubble term ranges over the chunks that exist on the
replica (a full chunk of bucket j only when m_j > 0, the remainder chunk only when r_j > 0);
t(0, s) = 0 (no chunk).  With every bucket holding at least one full chunk this is the
paper's max over j.
"""
from __future__ import annotations

from typing import Callable, Sequence


def schedule(d: Sequence[int], s: Sequence[int], M: int):
    """Per bucket (b_j, m_j, r_j) with d_j = m_j b_j + r_j, b_j = floor(M / s_j)."""
    out = []
    for dj, sj in zip(d, s):
        if sj < 1 or sj > M:
            raise ValueError(f"bucket length {sj} outside [1, M={M}]")
        bj = M // sj
        out.append((bj, dj // bj, dj % bj))
    return out


def replica_time(d: Sequence[int], s: Sequence[int], M: int, t: Callable[[int, int], float],
                 pp: int = 1) -> float:
    """App. D replica time: compute time + (pp - 1) x the longest chunk (1F1B bubble)."""
    if pp < 1:
        raise ValueError("pp >= 1")
    compute = 0.0
    longest = 0.0
    for (bj, mj, rj), sj in zip(schedule(d, s, M), s):
        full = t(bj, sj) if mj > 0 else 0.0
        rem = t(rj, sj) if rj > 0 else 0.0
        compute += mj * full + rem
        longest = max(longest, full, rem)
    return compute + (pp - 1) * longest


def fixed_length_time(b: int, s: int, m: int, t: Callable[[float, int], float], pp: int) -> float:
    """Eq. appendix_cost_model_pp_fixed_len: a mini-batch (b, s) split into m micro-batches."""
    return m * t(b / m, s) + (pp - 1) * t(b / m, s)


def quadratic_t(c0: float, c1: float, c2: float) -> Callable[[int, int], float]:
    """App. D's fitted t(b, s): "quadratic with respect to s and proportional to b",
    with the per-chunk constant of reading Q28: t = c0 + c1 b s + c2 b s^2 for b >= 1, 0 for b = 0."""
    return lambda b, s: 0.0 if b <= 0 else c0 + c1 * b * s + c2 * b * s * s
