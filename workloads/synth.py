"""Seeded synthetic workload generators (shared by tests, bench and smoke).

This module holds NO arithmetic of the method (no LoRA math, no bucketing, no
dispatch).  It only draws inputs: per-task sequence lengths shaped like the
paper's datasets (PAPER.md Table ``tb:dataset_summary``, lines 1098-1131), task
ids, adapter ranks/scales, and normally distributed tensor values.  Both the
oracle side (tests) and the CUDA side (bench, GPU tests) receive the SAME arrays
drawn here, so neither side ever generates inputs for the other.

Length model: each dataset's length distribution is a
lognormal fitted to the table's mean and skewness,
    (e^{s^2} + 2) * sqrt(e^{s^2} - 1) = skewness,   mu = ln(mean) - s^2 / 2,
truncated (clipped) to [16, L_max].  The resulting mixture is short-heavy with a
long tail, matching PAPER.md line 402 ("more than half of the sequences are
shorter than 2K, whilst only a few are longer than 8K").
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# (name, avg length, skewness, batch size)   -- PAPER.md lines 1106-1128
DATASETS = [
    ("dolly", 207, 7.11, 256),
    ("python_code", 269, 10.01, 128),
    ("Evol-Instruct", 702, 6.59, 128),
    ("CommitPackFt", 663, 0.79, 128),
    ("MathInstruct", 252, 3.03, 128),
    ("MetaMathQA", 236, 2.56, 128),
    ("NuminaMath-CoT", 543, 1.52, 256),
    ("PubMedQA", 371, 0.73, 64),
    ("XSum", 526, 7.49, 128),
    ("BillSum", 3903, 0.85, 32),
    ("cnn_dailymail", 947, 0.89, 256),
    ("MeetingBank", 3622, 4.35, 64),
]
_BY_NAME = {d[0]: d for d in DATASETS}


def lognormal_fit(mean: float, skew: float) -> tuple[float, float]:
    """(mu, sigma) of the lognormal with the given mean and skewness (bisection)."""
    def f(s):
        w = math.exp(s * s)
        return (w + 2.0) * math.sqrt(w - 1.0) - skew
    lo, hi = 1e-6, 3.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if f(mid) > 0:
            hi = mid
        else:
            lo = mid
    sigma = 0.5 * (lo + hi)
    mu = math.log(mean) - sigma * sigma / 2.0
    return mu, sigma


@dataclass
class TaskSpec:
    name: str
    mu: float
    sigma: float
    batch_size: int
    rank: int
    scale: float


@dataclass
class Workload:
    """A packed multi-task batch: per-sequence lengths and task ids plus adapter specs."""
    name: str
    tasks: list[TaskSpec]
    seq_lens: np.ndarray          # int32 [n]
    seq_task: np.ndarray          # int32 [n]
    l_max: int
    meta: dict = field(default_factory=dict)

    @property
    def T(self) -> int:
        return int(self.seq_lens.sum())

    @property
    def ranks(self) -> np.ndarray:
        return np.array([t.rank for t in self.tasks], dtype=np.int32)

    @property
    def scales(self) -> np.ndarray:
        return np.array([t.scale for t in self.tasks], dtype=np.float32)


def task_from_dataset(name: str, rank: int, scale: float, mean_scale: float = 1.0) -> TaskSpec:
    _, mean, skew, bs = _BY_NAME[name]
    mu, sigma = lognormal_fit(mean * mean_scale, skew)
    return TaskSpec(name, mu, sigma, bs, rank, scale)


def sample_lengths(rng: np.random.Generator, task: TaskSpec, n: int, l_min: int, l_max: int) -> np.ndarray:
    x = rng.lognormal(task.mu, task.sigma, size=n)
    return np.clip(np.rint(x), l_min, l_max).astype(np.int32)


def pack_tokens(tasks: list[TaskSpec], t_max: int, l_max: int, seed: int, l_min: int = 16,
                group_by_task: bool = True, name: str = "packed") -> Workload:
    """Draw sequences task-by-task (task chosen with probability proportional to its
    batch size, PAPER.md Table tb:dataset_summary 'Batch Size') until the packed token
    count reaches ``t_max``; the final sequence is shortened to fill exactly ``t_max``
    when that leaves >= l_min tokens.  Packing order is grouped by task (the order
    lobra_dispatch emits), stable in draw order within a task."""
    rng = np.random.default_rng(seed)
    w = np.array([t.batch_size for t in tasks], dtype=np.float64)
    w /= w.sum()
    lens, tids, total = [], [], 0
    while total < t_max:
        t = int(rng.choice(len(tasks), p=w))
        ln = int(sample_lengths(rng, tasks[t], 1, l_min, l_max)[0])
        if total + ln > t_max:
            ln = t_max - total
            if ln < l_min:
                break
        lens.append(ln)
        tids.append(t)
        total += ln
    lens = np.array(lens, dtype=np.int32)
    tids = np.array(tids, dtype=np.int32)
    if group_by_task:
        order = np.lexsort((np.arange(len(tids)), tids))
        lens, tids = lens[order], tids[order]
    return Workload(name, tasks, lens, tids, l_max, {"seed": seed, "t_max": t_max})


def sample_batch(tasks: list[TaskSpec], seed: int, l_max: int, l_min: int = 16,
                 per_task: list[int] | None = None) -> Workload:
    """One training step's global batch: ``batch_size`` sequences from every task
    (PAPER.md Table tb:dataset_summary batch sizes), in task order.  Used as the
    dispatch input (the batch before it is split across replicas)."""
    rng = np.random.default_rng(seed)
    lens, tids = [], []
    for t, spec in enumerate(tasks):
        n = spec.batch_size if per_task is None else per_task[t]
        lens.append(sample_lengths(rng, spec, n, l_min, l_max))
        tids.append(np.full(n, t, dtype=np.int32))
    return Workload("batch", tasks, np.concatenate(lens).astype(np.int32),
                    np.concatenate(tids).astype(np.int32), l_max, {"seed": seed})


# ----------------------------------------------------------------------------
# The BASELINE.json configs
# ----------------------------------------------------------------------------
LLAMA7B_PROJ = [  # (name, in, out)
    ("q", 4096, 4096), ("k", 4096, 4096), ("v", 4096, 4096), ("o", 4096, 4096),
    ("gate", 4096, 11008), ("up", 4096, 11008), ("down", 11008, 4096)]
LLAMA70B_PROJ = [
    ("q", 8192, 8192), ("k", 8192, 1024), ("v", 8192, 1024), ("o", 8192, 8192),
    ("gate", 8192, 28672), ("up", 8192, 28672), ("down", 28672, 8192)]


def config_c1(seed: int = 1) -> Workload:
    """C1 tiny: one 64x64 linear, 2 tasks r=4, s={2.0,0.5}, 8 sequences of length
    uniform in {3..40}, task ids alternating (fp32 path)."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(3, 41, size=8).astype(np.int32)
    tids = (np.arange(8) % 2).astype(np.int32)
    tasks = [TaskSpec("t0", 0, 0, 1, 4, 2.0), TaskSpec("t1", 0, 0, 1, 4, 0.5)]
    return Workload("C1", tasks, lens, tids, 40, {"seed": seed, "in": 64, "out": 64})


def c2_tasks() -> list[TaskSpec]:
    return [task_from_dataset(n, 16, 2.0) for n in ("dolly", "python_code", "Evol-Instruct", "MeetingBank")]


def config_c2(seed: int = 2, t_max: int = 16384) -> Workload:
    """C2: Llama-2-7B projections, 4 tasks r=16 s=2, lengths <= 4096, T = 16384."""
    w = pack_tokens(c2_tasks(), t_max, 4096, seed, name="C2")
    return w


def c3_tasks() -> list[TaskSpec]:
    names = [d[0] for d in DATASETS] + ["MeetingBank", "BillSum", "Evol-Instruct", "XSum"]
    ranks = [8, 16, 32, 64]
    scales = [0.5, 1.0, 2.0, 4.0]
    out = []
    for i, n in enumerate(names):
        t = task_from_dataset(n, ranks[i % 4], scales[i % 4])
        if i >= 12:
            t.name = n + "-like"
        out.append(t)
    return out


def config_c3(seed: int = 3, t_max: int = 65536) -> Workload:
    """C3: 16 tasks, ranks cycling 8/16/32/64, scales 0.5/1/2/4, lengths <= 16384, T = 65536."""
    return pack_tokens(c3_tasks(), t_max, 16384, seed, name="C3")


# ----------------------------------------------------------------------------
# Tensor values (numpy, host)
# ----------------------------------------------------------------------------
def normal(seed: int, shape, std: float = 1.0, dtype=np.float32) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(size=shape, dtype=np.float32) * np.float32(std)).astype(dtype)


def layer_tensors(wl: Workload, d_in: int, d_out: int, seed: int, zero_B: bool = False,
                  zero_W: bool = False) -> dict:
    """Host fp32 arrays for one projection: X [T,in], W [out,in], A_cat [sum r, in],
    B_cat [out, sum r], dY [T,out].  Distributions per SURVEY.md §8(d): X,dY ~ N(0,1);
    W, A ~ N(0,1/in); B_t ~ N(0,1/r_t)."""
    T = wl.T
    ranks = wl.ranks
    R = int(ranks.sum())
    X = normal(seed * 1000 + 1, (T, d_in))
    W = normal(seed * 1000 + 2, (d_out, d_in), 1.0 / math.sqrt(d_in))
    A = normal(seed * 1000 + 3, (R, d_in), 1.0 / math.sqrt(d_in))
    Bparts = []
    for t, r in enumerate(ranks):
        Bparts.append(normal(seed * 1000 + 10 + t, (d_out, int(r)), 1.0 / math.sqrt(int(r))))
    B = np.concatenate(Bparts, axis=1) if Bparts else np.zeros((d_out, 0), np.float32)
    dY = normal(seed * 1000 + 4, (T, d_out))
    if zero_B:
        B[:] = 0
    if zero_W:
        W[:] = 0
    return {"X": X, "W": W, "A": A, "B": B, "dY": dY}


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 -> fp32 (the values the bf16 path receives)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)
