"""GPU-seconds ablation of the paper's dispatch designs on B200 layer costs.

    python tools/ablation.py [--steps 20] [--out profiles/r1_ablation.json]     (under gpurun)

1. MEASURES the time of one Llama-2-7B layer's seven LoRA projections (fwd + bwd, C2 task
   mix, this library's kernels) on one B200 for packed chunks of T tokens, and fits
   t_1(T) = a0 + a1 * T (projection-only layers are linear in tokens: App. D's t(b, s) with
   no s^2 term).
2. MODELS a TP-k replica as t_k(T) = a0 + a1 * T / k + 4 all-reduces of T x 4096 bf16 at the
   measured 8-rank NCCL bus bandwidth (B200_PROFILING.md: 725 GB/s); Megatron TP.
3. For C5-like steps (the 12 dataset-table tasks + 4 clones, batch sizes of Table
   tb:dataset_summary, lengths <= 16K) on N = 8 GPUs with the per-replica token limits of
   DESIGN.md Q25 (TP1 8K, TP2 16K, TP4 32K), evaluates:
     A  Task-Fused: homogeneous replicas able to hold the longest sequence, uniform dispatch
     B  heterogeneous replicas + length-based dispatch (fixed 1K buckets)
     C  + workload-balanced dispatch (Eq. 3, fixed 1K buckets)
     D  + dynamic bucketing (256 grid, R = 16)  -- LobRA
   with every dispatch computed by lobra_dispatch (the exact C++ solver), the deployment
   for B-D chosen by enumerating all TP{1,2,4} mixes of 8 GPUs (a small stage-1 search).
GPU-seconds per step = N x max over replicas of the sum of its chunk times.

--padding: the paper's own setting ("we assume padding"): micro-batches of App. D
(chunking = 0: b_j = floor(M_i / s_j) sequences of bucket j, every sequence padded to s_j),
each chunk executed and charged at its PADDED tokens, and Eq. 3's per-sequence cost made
consistent with that execution: c_ij = t_i(s_j) + a0 / b_j (the per-chunk constant
amortised over a full micro-batch, App. D t(b, s) = a0 + b t(s)).  --r-sweep adds the
R-sensitivity study of P:1155-1161 (R = 4..32: padding tokens and step time of D).

--layer-cost profiles/r1_layer_cost.json (tools/bench_layer.py --fit) replaces step 1 by the
full decoder layer's measured App. D cost t = c0 + c1 sum(s) + c2 sum(s^2) per chunk
(attention's s^2 term real); TP-k replicas divide the token-dependent part
by k.  Output then goes to profiles/r1_ablation_layer.json.
"""
from __future__ import annotations

import argparse
import itertools
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_01193_b200 import _lib  # noqa: E402
from workloads import synth  # noqa: E402

M_LIMIT = {1: 8192, 2: 16384, 4: 32768}
BUS_BW = 725e9


def measure_layer(Ts=(1024, 2048, 4096, 8192, 16384), reps=5):
    import torch
    from paper_2509_01193_b200.layer import LLAMA2_7B, LoraLayer
    dev = torch.device("cuda:0")
    torch.cuda.set_device(0)
    tasks = synth.c2_tasks()
    layer = LoraLayer(LLAMA2_7B, [t.rank for t in tasks], [t.scale for t in tasks], dev, seed=1)
    io = layer.alloc_io(max(Ts), seed=2)
    out = {}
    for T in Ts:
        wl = synth.pack_tokens(tasks, T, 4096, seed=10 + T, name="cal")
        for _ in range(2):
            layer.forward(wl.seq_lens, wl.seq_task, io, T)
            layer.backward(wl.seq_lens, wl.seq_task, io, T, accumulate_dadb=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            layer.forward(wl.seq_lens, wl.seq_task, io, T)
            layer.backward(wl.seq_lens, wl.seq_task, io, T, accumulate_dadb=False)
        e1.record()
        torch.cuda.synchronize()
        out[T] = e0.elapsed_time(e1) / reps / 1000.0
    Tv = np.array(sorted(out), float)
    tv = np.array([out[int(T)] for T in Tv])
    a1, a0 = np.polyfit(Tv, tv, 1)
    return {"points_s": {int(k): v for k, v in out.items()}, "a0_s": float(a0), "a1_s_per_token": float(a1)}


QUAD = {"c2": 0.0}   # s^2 coefficient (seconds per token x length) when --layer-cost is given
PAD = {"on": False}  # --padding


def t_rep(k, T, a0, a1, S2=0.0):
    """Chunk time on a TP-k replica: T tokens, S2 = sum of squared sequence lengths."""
    comm = 0.0 if k == 1 else 4 * 2 * (k - 1) / k * T * 4096 * 2 / BUS_BW
    return a0 + (a1 * T + QUAD["c2"] * S2) / k + comm


def cost_table(groups, a0, a1, grid_step, grid_max, unit=1e-5):
    U = grid_max // grid_step
    out = []
    for tp, _, M in groups:
        row = []
        for u in range(U):
            sj = (u + 1) * grid_step
            c = t_rep(tp, sj, 0.0, a1, float(sj) ** 2)
            if PAD["on"]:
                c += a0 / max(1, M // sj)      # per-chunk constant over a full micro-batch
            row.append(max(1, int(round(c / unit))))
        out.append(row)
    return out


def step_time(groups, wl, mode, grid_step, R, a0, a1):
    tp = [g[0] for g in groups]
    reps = [g[1] for g in groups]
    M = [g[2] for g in groups]
    gmax = 16384
    d = _lib.lobra_dispatch(tp, reps, M, cost_table(groups, a0, a1, grid_step, gmax), wl.seq_lens,
                            wl.seq_task, grid_step, gmax, R, mode, chunking=0 if PAD["on"] else 1)
    rbase = np.concatenate([[0], np.cumsum(reps)])
    bnd = np.asarray(d["boundaries"], np.float64)
    times = []
    for rep in range(int(rbase[-1])):
        gi = int(np.searchsorted(rbase, rep, side="right") - 1)
        mine = d["seq_replica"] == rep
        t = 0.0
        for c in set(d["seq_chunk"][mine].tolist()):
            sel = mine & (d["seq_chunk"] == c)
            ls = wl.seq_lens[sel].astype(np.float64)
            if PAD["on"]:   # every sequence of an App. D micro-batch padded to its bucket length
                ls = bnd[d["seq_bucket"][sel]]
            t += t_rep(tp[gi], float(ls.sum()), a0, a1, float((ls ** 2).sum()))
        times.append(t)
    pad_tokens = float((bnd[d["seq_bucket"]] - wl.seq_lens).sum())
    return max(times), float(np.mean(times)), pad_tokens


def deployments(n=8, tps=(1, 2, 4)):
    """All (tp, replicas, M) mixes using exactly n GPUs, ordered by (tp, M)."""
    out = []
    for counts in itertools.product(*[range(n // t + 1) for t in tps]):
        if sum(c * t for c, t in zip(counts, tps)) == n:
            out.append([(t, c, M_LIMIT[t]) for c, t in zip(counts, tps) if c > 0])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_ablation.json"))
    ap.add_argument("--a0", type=float, default=None, help="skip the GPU measurement (seconds)")
    ap.add_argument("--a1", type=float, default=None)
    ap.add_argument("--layer-cost", default=None, help="App. D fit of the full layer (tools/bench_layer.py)")
    ap.add_argument("--padding", action="store_true", help="the paper's padded micro-batches (P:272)")
    ap.add_argument("--r-sweep", action="store_true", help="R-sensitivity of D (P:1155-1161)")
    ap.add_argument("--calibration", default=None, help="reuse the calibration of a previous ablation JSON")
    args = ap.parse_args()
    PAD["on"] = args.padding
    if args.layer_cost:
        lc = json.load(open(args.layer_cost))
        cal = {"source": args.layer_cost, "model": lc["model"], "a0_s": lc["c0_ms"] / 1e3,
               "a1_s_per_token": lc["c1_ms_per_token"] / 1e3, "c2_s_per_token_len": lc["c2_ms_per_token_len"] / 1e3}
        QUAD["c2"] = cal["c2_s_per_token_len"]
        if args.out.endswith("r1_ablation.json"):
            args.out = args.out.replace("r1_ablation.json", "r1_ablation_layer.json")
    elif args.calibration:
        cal = json.load(open(args.calibration))["calibration"]
    elif args.a0 is None:
        cal = measure_layer()
    else:
        cal = {"points_s": {}, "a0_s": args.a0, "a1_s_per_token": args.a1}
    a0, a1 = cal["a0_s"], cal["a1_s_per_token"]
    tasks = synth.c3_tasks()
    per_task = [t.batch_size for t in tasks[:12]] + [64] * 4
    batches = [synth.sample_batch(tasks, seed=100 + i, l_max=16384, per_task=per_task)
               for i in range(args.steps)]
    n = 8
    res = {"calibration": cal, "n_gpus": n, "steps": args.steps, "padding": PAD["on"], "strategies": {}}
    # A: Task-Fused, homogeneous TP able to hold the longest sequence of every batch
    longest = max(int(b.seq_lens.max()) for b in batches)
    tpA = min(t for t in (1, 2, 4) if M_LIMIT[t] >= longest)
    depA = [(tpA, n // tpA, M_LIMIT[tpA])]
    t0 = time.time()
    # the naive design fuses the batches with the same fixed 1K buckets as B and C (its padding
    # is what dynamic bucketing, D, removes)
    sA = [step_time(depA, b, 2, 1024, 16, a0, a1) for b in batches]
    res["strategies"]["A_task_fused"] = {"deployment": depA, "step_s": float(np.mean([x[0] for x in sA])),
                                         "pad_tokens": float(np.mean([x[2] for x in sA]))}
    # B-D on the best heterogeneous deployment for D (covering the longest sequence)
    best = None
    for dep in deployments(n):
        if max(g[2] for g in dep) < longest:
            continue
        sD = [step_time(dep, b, 0, 256, 16, a0, a1)[0] for b in batches[:5]]
        key = float(np.mean(sD))
        if best is None or key < best[0]:
            best = (key, dep)
    dep = best[1]
    for name, mode, grid in (("B_hetero_length_fixed", 1, 1024), ("C_hetero_balanced_fixed", 0, 1024),
                             ("D_lobra_balanced_dynamic", 0, 256)):
        st = [step_time(dep, b, mode, grid, 16, a0, a1) for b in batches]
        res["strategies"][name] = {"deployment": dep, "step_s": float(np.mean([x[0] for x in st])),
                                   "mean_replica_s": float(np.mean([x[1] for x in st])),
                                   "pad_tokens": float(np.mean([x[2] for x in st]))}
    base = res["strategies"]["A_task_fused"]["step_s"]
    for k, v in res["strategies"].items():
        v["gpu_seconds"] = n * v["step_s"]
        v["reduction_vs_task_fused"] = 1.0 - v["step_s"] / base
    if args.r_sweep:
        res["r_sweep"] = {}
        for R in (4, 8, 12, 16, 24, 32):
            st = [step_time(dep, b, 0, 256, R, a0, a1) for b in batches]
            res["r_sweep"][R] = {"step_s": float(np.mean([x[0] for x in st])),
                                 "pad_tokens": float(np.mean([x[2] for x in st])),
                                 "reduction_vs_task_fused": 1.0 - float(np.mean([x[0] for x in st])) / base}
    res["planning_wall_s"] = time.time() - t0
    res["tokens_per_step"] = float(np.mean([b.T for b in batches]))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
