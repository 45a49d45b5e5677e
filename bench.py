#!/usr/bin/env python
"""Benchmark of the LobRA multi-LoRA hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lobra|reference]
    python bench.py --plan-only            # CPU: the N = 1/2/4/8 deployments and dispatches

One STEP = one pass of the whole hot path over one batch:
per-step dispatch on the host (a7: bucketing DP + exact Eq. 3 + chunking), then for
every micro-batch of this rank's replica the forward and backward of all seven
Llama-2-7B projections with every task's adapters (a0-a5, TP collectives a6), then the
adapter-gradient all-reduce across replicas (a8).

N = 1 (default workload): BASELINE configs[2] = C3, the largest single-GPU configuration
(7B shapes, 16 tasks ranks 8-64, long-tail lengths <= 16K, T = 65536 packed, bf16, 1 x TP1);
a short C2 run (configs[1]) is reported beside it (`c2`).  N > 1 (torchrun, one rank per GPU):
C5 = weak scaling, N x 65536 tokens of the same 16-task mix per step, dispatched by Eq. 3 over
the heterogeneous deployment the stage-1 planner (lobra_plan_deployment) picks from TP1 /
TP2 / TP4 candidates with max tokens per chunk 8192 / 16384 / 32768 (Q25) and a
cost table built from measured per-TP layer timings (profiles/r2_tp_costs_7b.json, App. D
"offline profiling" P:1485; `--plan-only` prints the plans).

value = real tokens processed by all ranks / max-over-ranks device time (the whole-job
aggregate, as the bench contract asks; `per_gpu` = value / N).  Inputs are resident in HBM
when the timed region starts; every projection input exceeds L2 (>= 128 MiB per step-input
vs 126 MB L2), so no explicit L2 flush is used.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "multi-LoRA fwd+bwd tokens/s/GPU at 1/2/4/8 B200; % of bf16 tensor peak"
WORKLOAD_NAMES = {
    "c2": "C2 (BASELINE configs[1]): Llama-2-7B layer, 7 LoRA projections (q,k,v,o,gate,up,down), "
          "4 tasks r=16 s=2, lengths<=4096 packed, T=16384",
    "c3": "C3 (BASELINE configs[2]): Llama-2-7B layer, 7 LoRA projections (q,k,v,o,gate,up,down), "
          "16 tasks ranks 8/16/32/64 s 0.5-4, lengths<=16384 packed, T=65536",
    "c5": "C5 (BASELINE configs[4]): Llama-2-7B layer, 7 LoRA projections, C3's 16 tasks, N x 65536 tokens "
          "per step dispatched by Eq. 3 over the planner's heterogeneous TP1/TP2/TP4 replicas",
}
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML polled every 10 ms
    from a thread (the GPU found by its PCI bus id, so CUDA_VISIBLE_DEVICES remapping does
    not matter); `nvidia-smi -lms 100` when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.sm, self.mx, self.reasons = [], [], set()
        self.nvml = None
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            try:
                pr = torch.cuda.get_device_properties(gpu_index)
                bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
                h = nv.nvmlDeviceGetHandleByPciBusId_v2(bus)
            except Exception:
                h = nv.nvmlDeviceGetHandleByIndex(gpu_index)
            self.bits = [(n, getattr(nv, b)) for n, b in zip(self.NAMES, (
                "nvmlClocksEventReasonHwSlowdown", "nvmlClocksEventReasonHwThermalSlowdown",
                "nvmlClocksEventReasonSwThermalSlowdown", "nvmlClocksEventReasonSwPowerCap"))]
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.nvml, self.h = nv, h
        except Exception:
            self.nvml = None

    def _poll(self):
        nv, h = self.nvml, self.h
        while not self.stop_ev.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                self.mx.append(float(self.max_mhz))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for n, bit in self.bits:
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            self.stop_ev.wait(0.01)

    def start(self):
        if self.nvml is not None:
            self.stop_ev = threading.Event()
            self.th = threading.Thread(target=self._poll, daemon=True)
            self.th.start()
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.nvml is not None:
            self.stop_ev.set()
            self.th.join(timeout=5)
            src = "nvml 10 ms"
        elif self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        else:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            src = "nvidia-smi 100 ms"
            for ln in self.lines:
                parts = [x.strip() for x in ln.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    self.sm.append(float(parts[0]))
                    self.mx.append(float(parts[1]))
                except ValueError:
                    continue
                for nm, v in zip(self.NAMES, parts[4:8]):
                    if v.lower() == "active":
                        self.reasons.add(nm)
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else None, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": src}


# ------------------------------------------------------------------------------ plans
C5_CANDIDATES = [(1, 8192), (2, 16384), (4, 32768)]   # (TP degree, max tokens per chunk), Q25
C5_TOKENS_PER_GPU = 65536
GRID_MAX = 16384             # longest sequence of C3 / C5 (grid 256)
COST_UNIT_US = 10.0          # integer cost unit of the dispatch tables (reading Q15)
ALLREDUCE_GBS = 700.0        # assumed NVLink 5 all-reduce bus bandwidth


def tp_costs():
    """Per-token device time (us) of one Llama-2-7B layer's seven LoRA projections fwd+bwd on
    a TP-k replica: the measured per-rank shard compute (tools/bench_tp_shapes.py --model 7b
    --workload c3, profiles/r2_tp_costs_7b.json) plus the four T x h bf16 TP all-reduces per
    layer at ALLREDUCE_GBS (2 (k-1)/k of the message per rank, ring/two-shot volume)."""
    p = os.path.join(ROOT, "profiles", "r2_tp_costs_7b.json")
    comp = {1: 0.70, 2: 0.37, 4: 0.20, 8: 0.11}            # fallback: round-1 C3 scaling
    src = "fallback (round-1 C3 per-token time / TP)"
    if os.path.exists(p):
        d = json.load(open(p))
        comp = {int(k): float(v) for k, v in d["us_per_token"].items()}
        src = "measured (profiles/r2_tp_costs_7b.json)"
    out = {}
    for tp, us in comp.items():
        comm = 0.0 if tp == 1 else 4 * 4096 * 2 * 2 * (tp - 1) / tp / (ALLREDUCE_GBS * 1e3)
        out[tp] = us + comm
    return out, src


def cost_table(groups, grid_step=256, grid_max=32768):
    """Integer per-sequence cost c_i(u) on the grid (reading Q15): the projections are linear
    in tokens (App. D with a2 = 0 for projection-only layers), c = u * t_tp / unit."""
    per_tok, _ = tp_costs()
    U = grid_max // grid_step
    return [[max(1, int(round((k + 1) * grid_step * per_tok.get(tp, per_tok[1] / tp) / COST_UNIT_US)))
             for k in range(U)] for tp, _, _ in groups]


def c5_batch(n_gpus: int, step: int):
    from workloads import synth
    return synth.pack_tokens(synth.c3_tasks(), C5_TOKENS_PER_GPU * n_gpus, 16384, seed=1000 + step, name="C5")


def deployment_for(n_gpus: int):
    """(tp, replicas, max_tokens) per deployed group, ordered by (tp, M), chosen by the
    paper's stage-1 planner (lobra_plan_deployment: §4.2 Eq. 2 + App. A) on a sample of
    100 x B lengths of the step's task mix with the bench cost model.  N = 1 is
    C3's single TP1 replica (one chunk of the whole 65536-token batch)."""
    if n_gpus == 1:
        return [(1, 1, C5_TOKENS_PER_GPU)]
    from paper_2509_01193_b200 import _lib
    from workloads import synth
    tasks = synth.c3_tasks()
    per_step = c5_batch(n_gpus, 0).seq_lens
    sample = synth.sample_batch(tasks, seed=8, l_max=16384,
                                per_task=[max(1, 100 * len(per_step) * t.batch_size //
                                              sum(x.batch_size for x in tasks)) for t in tasks])
    cands = [(tp, 0, m) for tp, m in C5_CANDIDATES]
    res = _lib.lobra_plan_deployment([c[0] for c in cands], [c[2] for c in cands],
                                     cost_table(cands, 256, GRID_MAX), n_gpus, sample.seq_lens,
                                     len(per_step), 256, GRID_MAX, 16)
    groups = [(tp, int(p), m) for (tp, m), p in zip(C5_CANDIDATES, res["replicas"]) if p > 0]
    if sum(tp * p for tp, p, _ in groups) != n_gpus:
        raise SystemExit(f"planner deployment {groups} does not use all {n_gpus} GPUs")
    return groups


def plan_only():
    """CPU: print the deployment and the step-0 dispatch status / solve time per N."""
    from paper_2509_01193_b200 import _lib
    per_tok, src = tp_costs()
    for n in (1, 2, 4, 8):
        groups = deployment_for(n)
        wl = c5_batch(n, 0) if n > 1 else None
        line = {"n_gpus": n, "deployment": "+".join(f"{p}xTP{tp}(M={m})" for tp, p, m in groups),
                "us_per_token": per_tok, "cost_source": src}
        if wl is not None:
            t0 = time.perf_counter()
            d = _lib.lobra_dispatch([g[0] for g in groups], [g[1] for g in groups], [g[2] for g in groups],
                                    cost_table(groups, 256, GRID_MAX), wl.seq_lens, wl.seq_task, 256, GRID_MAX,
                                    16, 0, chunking=1)
            line.update({"status": d["status"], "t_hat": d["t_hat"], "solve_ms": 1000 * (time.perf_counter() - t0),
                         "num_seqs": int(len(wl.seq_lens)), "tokens": int(wl.seq_lens.sum()),
                         "nodes": d["nodes"]})
        print(json.dumps(line), flush=True)


def replica_ranks(groups):
    """Global replica id -> list of ranks (contiguous, group-major)."""
    out, r = [], 0
    for tp, p, _ in groups:
        for _ in range(p):
            out.append(list(range(r, r + tp)))
            r += tp
    return out


# ------------------------------------------------------------------------------ oracle leg
def oracle_tokens_per_s(wl, shapes, budget_tokens=2048, seed=7):
    """The fp64 CPU oracle (test infrastructure) timed on the host cores on a bounded
    sample of the workload: the first sequences of the batch totalling ~budget_tokens,
    all seven projections forward + backward."""
    from oracle import lora as O
    from workloads import synth
    lens, tasks, tot = [], [], 0
    for L, t in zip(wl.seq_lens.tolist(), wl.seq_task.tolist()):
        if tot >= budget_tokens:
            break
        L = min(L, budget_tokens - tot)
        lens.append(L)
        tasks.append(t)
        tot += L
    sub = synth.Workload("sample", wl.tasks, np.array(lens, np.int32), np.array(tasks, np.int32), wl.l_max)
    data = []
    for i, (_, d_in, d_out, _, _) in enumerate(shapes):
        t = synth.layer_tensors(sub, d_in, d_out, seed=seed + i)
        data.append({k: synth.round_bf16(v).astype(np.float64) for k, v in t.items()})
    t0 = time.perf_counter()
    for t in data:
        args = (t["X"], t["W"], t["A"], t["B"], sub.ranks.tolist(), sub.scales, sub.seq_lens, sub.seq_task)
        O.lora_fwd(*args)
        O.lora_bwd(*args, t["dY"])
    dt = time.perf_counter() - t0
    threads = os.cpu_count()
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 0) for i in threadpool_info()] + [1])
    except Exception:
        pass
    return tot / dt, dt, tot, threads


def run_reference(args):
    """--impl reference: the oracle (as it stands) on the host cores, bounded samples of
    the same workload as the lobra arm (C3 at N = 1, C5 at N > 1); rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2509_01193_b200.layer import LLAMA2_7B
    from workloads import synth
    workload = args.workload or ("c3" if args.gpus == 1 else "c5")
    wl = {"c2": lambda: synth.config_c2(), "c3": lambda: synth.config_c3(),
          "c5": lambda: c5_batch(args.gpus, 0)}[workload]()
    budget = 2048
    times, toks = [], 0
    for i in range(args.warmup + args.steps):
        tps, dt, n, threads = oracle_tokens_per_s(wl, LLAMA2_7B, budget_tokens=budget, seed=100 + i)
        if i >= args.warmup:
            times.append(dt)
            toks = n
    tot = sum(times)
    value = toks * len(times) / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * tot / len(times), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD_NAMES[workload], "global_batch_tokens": toks, "parallelism": "host"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "oracle",
                             "sample": f"first {toks} tokens of the {workload.upper()} batch, 7 projections "
                                       "fwd+bwd, fp64 NumPy"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def c2_side(args):
    """N = 1: the C2 configuration (BASELINE configs[1]) measured beside the C3 headline, in
    a fresh process (same timing rules, no e2e / oracle legs)."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "c2", "--steps", str(args.steps),
           "--warmup", str(args.warmup), "--no-e2e", "--no-cpu", "--no-c2"]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        d = json.loads(r.stdout.strip().splitlines()[-1])
        return {k: d[k] for k in ("value", "unit", "ms_per_step", "algorithmic_tflops", "frac_of_bf16_peak",
                                  "roofline", "clocks", "gpu_launches")} | {"workload": d["config"]["workload"]}
    except Exception as e:   # reported, never fatal for the headline line
        return {"error": str(e)[:200]}


# ------------------------------------------------------------------------------ main leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lobra", choices=["lobra", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="few steps, no e2e/cpu (for ncu)")
    ap.add_argument("--workload", default="", choices=["", "c2", "c3", "c5"],
                    help="default: c3 at N = 1 (BASELINE configs[2], the largest single-GPU config), c5 at "
                         "N > 1 (weak scaling over heterogeneous replicas); c2 = configs[1] (N = 1)")
    ap.add_argument("--no-c2", action="store_true", help="N = 1: skip the C2 side measurement")
    ap.add_argument("--plan-only", action="store_true", help="CPU: print the N = 1/2/4/8 plans and exit")
    ap.add_argument("--no-kernel-events", action="store_true",
                    help="do not record per-kernel CUDA events inside the timed region")
    args = ap.parse_args()
    lobra_env = {k: v for k, v in sorted(os.environ.items()) if k.startswith("LOBRA_")}
    dbg = [k for k in lobra_env if k.startswith("LOBRA_DBG_") or k == "LOBRA_META_CACHE"]
    if dbg:   # work-skipping probes (compiled only with -DLOBRA_PROBES): never a bench number
        raise SystemExit(f"bench.py refuses to run with probe variables set: {', '.join(dbg)}")
    if args.plan_only:
        return plan_only()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2509_01193_b200 import _lib
    from paper_2509_01193_b200.layer import LLAMA2_7B, LoraLayer, algorithmic_flops
    from workloads import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n_gpus = max(world, 1)
    # LOBRA_BENCH_GLOO=1: test mode for the N > 1 control flow on ONE GPU (all ranks share
    # cuda:0, gloo process group, TP1 replicas only, adapter sync through torch.distributed)
    gloo_test = os.environ.get("LOBRA_BENCH_GLOO") == "1"
    if gloo_test:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if gloo_test:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    _lib.load()

    workload = args.workload or ("c3" if n_gpus == 1 else "c5")
    if workload in ("c2", "c3") and n_gpus > 1:
        raise SystemExit(f"--workload {workload} is a single-GPU configuration (use c5 for N > 1)")
    if workload == "c5" and gloo_test:
        groups = [(1, n_gpus, C5_TOKENS_PER_GPU)]
    elif workload == "c5":
        groups = deployment_for(n_gpus)
    else:
        groups = [(1, 1, C5_TOKENS_PER_GPU if workload == "c3" else 16384)]
    reps = replica_ranks(groups)
    my_rep = next(i for i, rr in enumerate(reps) if rank in rr)
    my_group = 0
    acc = 0
    for gi, (tp, p, _) in enumerate(groups):
        if my_rep < acc + p:
            my_group = gi
            break
        acc += p
    tp_size = groups[my_group][0]
    tp_rank = reps[my_rep].index(rank)
    comm = None
    if world > 1 and not gloo_test:
        uid = [_lib.lobra_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = _lib.lobra_comm_init(uid[0], world, rank, my_rep)

    # TP all-reduces through the library's own peer-memory collective (lobra_symm_*: CUDA IPC
    # buffers over NVLink) unless LOBRA_TP_COLLECTIVE=nccl; NCCL if any rank fails
    # to set it up.  Handles travel over the world process group; every rank takes part.
    symm = None
    any_tp = any(g[0] > 1 for g in groups)
    tp_coll = "nccl" if any_tp else "none"
    if comm is not None and os.environ.get("LOBRA_TP_COLLECTIVE", "own") != "nccl":
        mine, err = None, ""
        if tp_size > 1:
            try:
                symm = _lib.Symm(tp_rank, tp_size, groups[my_group][2] * 4096 * 2)
                mine = symm.handle
            except Exception as e:   # setup failure -> NCCL on every rank
                err = str(e)
        allh = [None] * world
        dist.all_gather_object(allh, (mine, err))
        ok = all(not e for _, e in allh)
        if ok and symm is not None:
            try:
                symm.open([allh[r][0] for r in reps[my_rep]])
            except Exception:
                ok = False
        flag = torch.tensor([1 if ok else 0], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 1 and any_tp:
            tp_coll = "own (CUDA IPC peer memory, two-shot, lobra_symm)"
        if int(flag.item()) == 1 and symm is not None:
            _lib.lobra_comm_attach_symm(comm, symm)
        elif symm is not None:
            symm.destroy()
            symm = None

    tasks = synth.c2_tasks() if workload == "c2" else synth.c3_tasks()
    ranks = [t.rank for t in tasks]
    scales = [t.scale for t in tasks]
    layer = LoraLayer(LLAMA2_7B, ranks, scales, dev, torch.bfloat16, tp_size, tp_rank, comm, seed=1234,
                      group_inputs=os.environ.get("LOBRA_NO_GROUPS") != "1")
    max_tok = groups[my_group][2]
    io = layer.alloc_io(max_tok, seed=99 + rank)

    tp_list = [g[0] for g in groups]
    rep_list = [g[1] for g in groups]
    m_list = [g[2] for g in groups]
    grid_step, grid_max = 256, GRID_MAX if workload != "c2" else 4096
    costs = cost_table(groups, grid_step, grid_max)

    def make_batch(step: int):
        """Global batch of the step (seeded): C3 / C2 at N = 1, N x 65536 tokens of the C3
        task mix at N > 1 (C5)."""
        if workload == "c3":
            return synth.config_c3(seed=3 + step)
        if workload == "c2":
            return synth.config_c2(seed=2 + step)
        return c5_batch(n_gpus, step)

    n_batches = 4
    batches = [make_batch(i) for i in range(n_batches)]

    def plan(wl):
        # raises on LOBRA_ERR_BUDGET: a bench step never runs a non-Eq.-3 dispatch
        d = _lib.lobra_dispatch(tp_list, rep_list, m_list, costs, wl.seq_lens, wl.seq_task,
                                grid_step, grid_max, 16, 0, chunking=1)
        assert d["status"] == 0
        mine = np.nonzero(d["seq_replica"] == my_rep)[0]
        chunks = []
        for c in sorted(set(d["seq_chunk"][mine].tolist())):
            idx = mine[d["seq_chunk"][mine] == c]
            idx = idx[np.argsort(d["pack_order"][idx])]
            chunks.append((wl.seq_lens[idx].astype(np.int32), wl.seq_task[idx].astype(np.int32)))
        return chunks, int(wl.seq_lens.sum()), d

    def run_step(chunks, stream=None):
        if tp_size > 1:
            layer.flat_grad.zero_()
        for ci, (lens, tsk) in enumerate(chunks):
            T = int(lens.sum())
            layer.forward(lens, tsk, io, T, stream=stream)
            layer.backward(lens, tsk, io, T, accumulate_dadb=(ci > 0 or tp_size > 1), stream=stream)
        if not chunks:   # a replica without work this step contributes zeros (P:170 sync)
            layer.flat_grad.zero_()
        if gloo_test and world > 1:
            dist.all_reduce(layer.flat_grad)
        else:
            layer.sync_adapter_grads(stream=stream)

    plans = [plan(b) for b in batches]
    stream = torch.cuda.current_stream()
    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(max_workers=1)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        run_step(plans[i % n_batches][0])
    barrier()

    peaks, peak_src = load_peaks()

    def timed(kernel_events=False):
        sampler = ClockSampler(local) if rank == 0 else None
        if sampler:
            sampler.start()
        _lib.lobra_profile_enable(kernel_events)
        _lib.lobra_profile_read(reset=True)
        l0 = _lib.lobra_launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tokens = 0
        tokens_local = 0
        disp_ms = []
        barrier()
        e0.record(stream)
        # a7: every step's dispatch is computed on the host one step ahead, in a worker thread
        # (the C++ call releases the GIL), while the GPU works on the enqueued step (P:586
        # "fast and can be fully overlapped by the training of previous step(s)")
        def timed_plan(b):
            t0 = time.perf_counter()
            r = plan(b)
            return r, 1000 * (time.perf_counter() - t0)
        fut = pool.submit(timed_plan, batches[args.warmup % n_batches])
        for i in range(args.steps):
            (chunks, tok, _), dms = fut.result()
            disp_ms.append(dms)
            if i + 1 < args.steps:
                fut = pool.submit(timed_plan, batches[(args.warmup + i + 1) % n_batches])
            run_step(chunks)
            tokens += tok
            tokens_local += sum(int(c[0].sum()) for c in chunks)
        e1.record(stream)
        torch.cuda.synchronize()
        ms_local = e0.elapsed_time(e1)
        launches = _lib.lobra_launch_count() - l0
        prof = _lib.lobra_profile_read(reset=True)
        _lib.lobra_profile_enable(False)
        clocks = sampler.stop() if sampler else None
        if world > 1:
            t = torch.tensor([ms_local], device="cpu" if gloo_test else dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_total = float(t.item())
        else:
            ms_total = ms_local
        return ms_total, ms_local, tokens, tokens_local, disp_ms, launches, prof, clocks

    def rejected(c):
        """hw/thermal slowdown, or SM clocks well below max with no reason (a clock lock)."""
        if not c or not c.get("sm_mhz") or not c.get("sm_max_mhz"):
            return False
        bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
        if bad & set(c["reasons"]):
            return True
        return c["sm_mhz"] < 0.85 * c["sm_max_mhz"] and not c["reasons"]

    # The official timed region runs uninstrumented: a CUDA event recorded between two launches
    # breaks their programmatic dependent launch (measured: ~0.3 ms per step with events around
    # all 35 launches).  A second pass over the same K steps records per-launch CUDA events on
    # the launching stream for the roofline and the per-class split (`roofline_pass`).
    ms_total, ms_local, tokens, tokens_local, disp_ms, launches, prof, clocks = timed()
    redo = [1 if (rank == 0 and rejected(clocks)) else 0]
    if world > 1:
        t = torch.tensor(redo, device="cpu" if gloo_test else dev)
        dist.broadcast(t, 0)
        redo = [int(t.item())]
    remeasured = None
    if redo[0]:
        remeasured = clocks
        ms_total, ms_local, tokens, tokens_local, disp_ms, launches, prof, clocks = timed()
    ms_step = ms_total / args.steps
    value = tokens / (ms_total / 1000.0)
    rf = {"pass": "none (--no-kernel-events)"}
    if not args.no_kernel_events and not args.profile_only:
        # idle gap so the instrumented pass starts from the same thermal / power state as the
        # official one (which follows the short warm-up); otherwise it runs at lower clocks
        barrier()
        time.sleep(2.0)
        barrier()
        for i in range(args.warmup):
            run_step(plans[i % n_batches][0])
        barrier()
        _, ms_local_ev, _, _, _, _, prof, clocks_ev = timed(kernel_events=True)
        rf = {"pass": "second pass over the same K steps with per-launch CUDA events on the launching "
                      "stream (events between launches disable programmatic dependent launch)",
              "ms_per_step": ms_local_ev / args.steps, "clocks": clocks_ev}
        ms_local = ms_local_ev

    # ---- roofline of the dominant kernel (device time share inside the timed region)
    T_step_local = tokens_local / args.steps
    # algorithmic FLOPs per GEMM class over the timed region (this rank's shards)
    fl_fwd = fl_bwd = 0.0
    nt = np.zeros(len(ranks))
    for i in range(args.steps):
        for lens, tsk in plan(batches[(args.warmup + i) % n_batches])[0]:
            for L, t in zip(lens.tolist(), tsk.tolist()):
                nt[t] += L
    tok_r = float((nt * np.array(ranks)).sum())
    for p in layer.projs:
        fl_fwd += 2.0 * nt.sum() * p.in_l * p.out_l + 2.0 * tok_r * p.out_l
        fl_bwd += 2.0 * nt.sum() * p.in_l * p.out_l + 2.0 * tok_r * p.in_l
    kern = {k: {"launches": c, "ms": ms} for k, (c, ms) in prof.items() if c}
    dom = max(("gemm_fwd", "gemm_bwd"), key=lambda k: prof[k][1])
    clocks = clocks if clocks is not None else {}
    dom_fl = fl_fwd if dom == "gemm_fwd" else fl_bwd
    dom_ms = prof[dom][1]
    # Peak: the task's rule -- the burst figure for a kernel timed alone, the SUSTAINED one
    # for a kernel timed inside a long step.  The dominant GEMM is timed inside the
    # multi-second C3 step (the roofline pass below), where the 1000 W cap holds the clock,
    # so the denominator is MEASURED_PEAKS' sustained cuBLAS throughput (back to back for 4 s
    # under the same cap); the burst ratio is reported beside as `frac_vs_burst`.
    capped = bool(clocks and "sw_power_cap" in clocks.get("reasons", []))
    peak_burst = float(peaks["bf16_tflops"])
    peak_kind = "bf16_tflops_sustained" if "bf16_tflops_sustained" in peaks else "bf16_tflops"
    peak_t = float(peaks[peak_kind])
    achieved = dom_fl / (dom_ms / 1000.0) / 1e12 if dom_ms > 0 else 0.0
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):   # ncu DRAM bytes per launch of this workload's dominant class
        traffic = json.load(open(tf)).get(workload, {}).get("k_gemm_" + dom.split("_")[1])
    # algorithmic DRAM bytes per launch of the class: each operand once (activations, the
    # weight, the bf16 output), averaged over the projections' launches
    Tl = T_step_local
    alg_b = float(np.mean([2.0 * (Tl * p.in_l + p.in_l * p.out_l + Tl * p.out_l) for p in layer.projs]))
    roofline = {"bound": "tensor", "kernel": f"k_gemm ({dom})", "achieved": achieved, "peak": peak_t,
                "algorithmic_bytes_per_launch": alg_b,
                "unit": "TFLOP/s", "frac": achieved / peak_t, "traffic": traffic,
                "peak_source": f"{peak_src} {peak_kind} (the kernel is timed inside a long step)" +
                               ("; sw_power_cap was active in the timed region" if capped else ""),
                "frac_vs_burst": achieved / peak_burst,
                "share_of_step": dom_ms / ms_local if ms_local > 0 else 0.0,
                "flops_per_launch": dom_fl / max(prof[dom][0], 1),
                "ms_per_launch": dom_ms / max(prof[dom][0], 1), "roofline_pass": rf}
    flops_step = algorithmic_flops(LLAMA2_7B, int(tokens / args.steps), ranks,
                                   tokens_per_task=(nt / args.steps).tolist())["total"]
    step_tflops = flops_step / (ms_step / 1000.0) / 1e12

    # ---- end to end through the public API with host buffers (pinned), rank-local
    e2e = None
    if not args.no_e2e and not args.profile_only:
        # End to end through the public API with HOST inputs: every micro-batch's X (4 input
        # groups) and dY (7 projections) come from pinned host memory and every step's
        # adapter gradients go back to the host.  The H2D copies of micro-batch k+1 run on a
        # copy stream while micro-batch k computes (double-buffered device inputs).
        host_x = {g: torch.empty(io["X"][g].shape, dtype=io["X"][g].dtype, pin_memory=True) for g in io["X"]}
        host_dy = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in io["dY"].items()}
        for g in host_x:
            host_x[g].copy_(io["X"][g])
        for k in host_dy:
            host_dy[k].copy_(io["dY"][k])
        host_grad = torch.empty(layer.flat_grad.shape, dtype=torch.float32, pin_memory=True)
        io2 = {"X": {g: torch.empty_like(v) for g, v in io["X"].items()},
               "dY": {k: torch.empty_like(v) for k, v in io["dY"].items()},
               "Y": io["Y"], "dX": io["dX"]}
        bufs = [io, io2]
        ke = max(1, min(args.steps, 5))
        items = []                                    # (step, lens, tasks, last_of_step)
        e2e_tokens = 0
        for i in range(ke):
            chunks, tok, _ = plan(batches[i % n_batches])
            e2e_tokens += tok
            for ci, (lens, tsk) in enumerate(chunks):
                items.append((i, lens, tsk, ci == len(chunks) - 1))
        h2d = d2h = 0
        # NC copy streams (LOBRA_E2E_COPY_STREAMS, default 2): the H2D tensors of a micro-batch
        # are spread over them so that several copy engines share the PCIe link
        nc = max(1, int(os.environ.get("LOBRA_E2E_COPY_STREAMS", "2")))
        comp = stream
        copy_ss = [torch.cuda.Stream(device=dev) for _ in range(nc)]
        ready = [[torch.cuda.Event() for _ in range(nc)] for _ in range(2)]
        free = [torch.cuda.Event() for _ in range(2)]
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(comp)
        for cs in copy_ss:
            cs.wait_event(f0)

        def issue_copy(k):
            nonlocal h2d
            b = k % 2
            T = int(items[k][1].sum())
            jobs = [(bufs[b]["X"][g], host_x[g]) for g in host_x] + \
                   [(bufs[b]["dY"][kk], host_dy[kk]) for kk in host_dy]
            jobs.sort(key=lambda j: -j[1][:T].numel())
            load = [0] * nc
            for ci, cs in enumerate(copy_ss):
                if k >= 2:
                    cs.wait_event(free[b])
            for dst, src in jobs:                    # largest first onto the least loaded stream
                ci = load.index(min(load))
                n = src[:T].numel() * src.element_size()
                load[ci] += n
                with torch.cuda.stream(copy_ss[ci]):
                    dst[:T].copy_(src[:T], non_blocking=True)
                h2d += n
            for ci, cs in enumerate(copy_ss):
                ready[b][ci].record(cs)

        trace = os.environ.get("LOBRA_E2E_TRACE") == "1"   # per-item event timeline on stderr
        tev = []
        if items:
            issue_copy(0)
        for k, (step_i, lens, tsk, last) in enumerate(items):
            if k + 1 < len(items):
                issue_copy(k + 1)
            b = k % 2
            for ev in ready[b]:
                comp.wait_event(ev)
            if trace:
                e = torch.cuda.Event(enable_timing=True)
                e.record(comp)
                tev.append(("start", k, e))
            T = int(lens.sum())
            first_of_step = k == 0 or items[k - 1][0] != step_i
            if first_of_step and tp_size > 1:
                layer.flat_grad.zero_()
            layer.forward(lens, tsk, bufs[b], T, stream=comp)
            layer.backward(lens, tsk, bufs[b], T, accumulate_dadb=not first_of_step or tp_size > 1,
                           stream=comp)
            free[b].record(comp)
            if last:
                if gloo_test and world > 1:
                    dist.all_reduce(layer.flat_grad)
                else:
                    layer.sync_adapter_grads(stream=comp)
                host_grad.copy_(layer.flat_grad, non_blocking=True)
                d2h += layer.flat_grad.numel() * 4
            if trace:
                e = torch.cuda.Event(enable_timing=True)
                e.record(comp)
                tev.append(("end", k, e))
        f1.record(comp)
        torch.cuda.synchronize()
        e_ms = f0.elapsed_time(f1)
        if trace:
            print(json.dumps({"e2e_trace_ms": [(w, k, round(f0.elapsed_time(e), 1)) for w, k, e in tev],
                              "total_ms": round(e_ms, 1)}), file=sys.stderr)
        if world > 1:
            t = torch.tensor([e_ms], device="cpu" if gloo_test else dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": e2e_tokens / (e_ms / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": int(h2d // ke), "d2h_bytes_per_step": int(d2h // ke),
               "steps": ke, "overlap": f"H2D of micro-batch k+1 on {nc} copy stream(s) during micro-batch k"}

    cpu = None
    if rank == 0 and n_gpus == 1 and not args.no_cpu and not args.profile_only:
        tps, dt, n, threads = oracle_tokens_per_s(batches[0], LLAMA2_7B, budget_tokens=8192)
        cpu = {"value": tps, "unit": "tokens/s", "cores": threads, "kind": "oracle",
               "sample": f"first {n} tokens of the {workload.upper()} batch, 7 projections fwd+bwd, "
                         f"fp64 NumPy ({dt:.1f} s)"}

    if rank == 0:
        par = "+".join(f"{p}xTP{tp}" for tp, p, _ in groups)
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": n_gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (seeded; lengths lognormal-fitted to the paper's dataset table)",
                "config": {"workload": WORKLOAD_NAMES[workload],
                           "global_batch_tokens": int(tokens / args.steps), "seq_len_max": grid_max,
                           "parallelism": par, "l2": "inputs > L2 (each projection input >= 128 MiB)",
                           "dispatch": "Eq. 3 exact (lobra_dispatch mode 0), packed chunks <= M_i tokens",
                           "cost_table": tp_costs()[1],
                           "tp_collective": tp_coll},
                "per_gpu": value / n_gpus,
                "algorithmic_tflops": step_tflops,
                "frac_of_bf16_peak": {"burst": step_tflops / float(peaks["bf16_tflops"]),
                                      "sustained": step_tflops / float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])),
                "nominal_2250": step_tflops / 2250.0},
                "clocks": clocks, **({"remeasured_after": remeasured} if remeasured else {}), "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline,
                "kernels": kern, "dispatch_ms_median": statistics.median(disp_ms) if disp_ms else None,
                "cpu_baseline": cpu, "lobra_env": lobra_env}
        if workload == "c3" and n_gpus == 1 and not args.no_c2 and not args.profile_only:
            line["c2"] = c2_side(args)
        print(json.dumps(line), flush=True)
    if comm is not None:
        torch.cuda.synchronize()
        comm.destroy()
    if world > 1:
        dist.barrier()
    if symm is not None:          # after every peer stopped using the mapped buffers
        symm.destroy()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
