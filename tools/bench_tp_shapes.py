"""Per-rank compute of TP-sharded Llama-2 projections on one B200 (run under gpurun).

Default: BASELINE config 4 (Llama-2-70B projections at TP 1/2/4/8, C2 batch T = 16384, 4
tasks r = 16).  `--model 7b --workload c3 --chunk 8192,16384,32768`: the per-TP costs of the
C5 deployments (Llama-2-7B, C3 task mix, one chunk per TP degree at its max tokens M =
8192 / 16384 / 32768, Q25) that bench.py's cost table is built from
(profiles/r2_tp_costs_7b.json, App. D "offline profiling").  Every rank of a TP group
runs its shard's GEMMs and LoRA kernels on the full micro-batch; this measures that local
compute (the TP all-reduces are excluded: one GPU here).  Column-parallel
q/k/v/gate/up keep `in` and shard `out`, row-parallel o/down shard `in` (Megatron).

    python tools/bench_tp_shapes.py [--steps 10] > profiles/<tag>_tp_shapes.jsonl
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def shard_shapes(shapes, tp):
    out = []
    for name, d_in, d_out, kind, group in shapes:
        if kind == "col":
            out.append((name, d_in, d_out // tp, "col", group))
        else:
            out.append((name, d_in // tp, d_out, "row", group))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--model", default="70b", choices=["7b", "70b"])
    ap.add_argument("--workload", default="c2", choices=["c2", "c3"])
    ap.add_argument("--tps", default="1,2,4,8")
    ap.add_argument("--chunk", default="", help="per-TP chunk tokens (comma list), default the whole batch")
    args = ap.parse_args()
    import torch
    from paper_2509_01193_b200 import _lib
    from paper_2509_01193_b200.layer import LLAMA2_7B, LLAMA2_70B, LoraLayer, algorithmic_flops
    from workloads import synth
    dev = torch.device("cuda:0")
    _lib.load()
    tasks = synth.c2_tasks() if args.workload == "c2" else synth.c3_tasks()
    ranks, scales = [t.rank for t in tasks], [t.scale for t in tasks]
    base = LLAMA2_70B if args.model == "70b" else LLAMA2_7B
    tps = [int(x) for x in args.tps.split(",")]
    chunks = [int(x) for x in args.chunk.split(",")] if args.chunk else [0] * len(tps)
    for tp, chunk in zip(tps, chunks):
        if args.workload == "c2":
            wl = synth.config_c2() if not chunk else synth.config_c2(t_max=chunk)
        else:
            wl = synth.config_c3() if not chunk else synth.pack_tokens(tasks, chunk, min(16384, chunk), seed=3,
                                                                      name="C3chunk")
        lens, tsk, T = wl.seq_lens.astype(np.int32), wl.seq_task.astype(np.int32), wl.T
        shapes = shard_shapes(base, tp)
        layer = LoraLayer(shapes, ranks, scales, dev, torch.bfloat16, 1, 0, None, seed=1234)
        io = layer.alloc_io(T, seed=99)

        def step():
            layer.forward(lens, tsk, io, T)
            layer.backward(lens, tsk, io, T, accumulate_dadb=False)

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        _lib.lobra_profile_enable(True)
        _lib.lobra_profile_read(reset=True)
        for _ in range(args.steps):
            step()
        prof = _lib.lobra_profile_read(reset=True)
        _lib.lobra_profile_enable(False)
        fl = algorithmic_flops(shapes, T, ranks)["total"]
        line = {"metric": f"Llama-2-{args.model.upper()} projections fwd+bwd, per-rank shard compute",
                "model": args.model, "workload": args.workload, "tokens": T,
                "tp": tp, "value": T / (ms / 1000.0), "unit": "tokens/s per rank", "ms_per_step": ms,
                "algorithmic_tflops": fl / (ms / 1000.0) / 1e12,
                "shapes": [f"{n} {i}->{o} ({k})" for n, i, o, k, _ in shapes],
                "ms_by_class": {k: v[1] / args.steps for k, v in prof.items() if v[0]},
                "note": "TP all-reduces excluded (one GPU); tokens/s of the TP group = this value",
                "dtype": "bf16", "data": f"synthetic {args.workload.upper()} batch (T={T})"}
        print(json.dumps(line), flush=True)
        del layer, io
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
