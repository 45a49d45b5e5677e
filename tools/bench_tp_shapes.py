"""Per-rank compute of BASELINE config 4 (Llama-2-70B projections TP-sharded at TP 1/2/4/8) on
one B200 (run under gpurun).  Every rank of a TP group runs its shard's GEMMs and LoRA kernels
on the full micro-batch; this measures that local compute (the TP all-reduces are excluded:
one GPU here).  Column-parallel q/k/v/gate/up keep `in` and shard `out`,
row-parallel o/down shard `in` (Megatron).  C2 batch (T = 16384, 4 tasks r = 16).

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
    args = ap.parse_args()
    import torch
    from paper_2509_01193_b200 import _lib
    from paper_2509_01193_b200.layer import LLAMA2_70B, LoraLayer, algorithmic_flops
    from workloads import synth
    dev = torch.device("cuda:0")
    _lib.load()
    tasks = synth.c2_tasks()
    ranks, scales = [t.rank for t in tasks], [t.scale for t in tasks]
    wl = synth.config_c2()
    lens, tsk, T = wl.seq_lens.astype(np.int32), wl.seq_task.astype(np.int32), wl.T
    for tp in (1, 2, 4, 8):
        shapes = shard_shapes(LLAMA2_70B, tp)
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
        line = {"metric": "Llama-2-70B projections fwd+bwd, per-rank shard compute (BASELINE config 4)",
                "tp": tp, "value": T / (ms / 1000.0), "unit": "tokens/s per rank", "ms_per_step": ms,
                "algorithmic_tflops": fl / (ms / 1000.0) / 1e12,
                "shapes": [f"{n} {i}->{o} ({k})" for n, i, o, k, _ in shapes],
                "ms_by_class": {k: v[1] / args.steps for k, v in prof.items() if v[0]},
                "note": "TP all-reduces excluded (one GPU); tokens/s of the TP group = this value",
                "dtype": "bf16", "data": "synthetic C2 batch (T=16384, 4 tasks r=16)"}
        print(json.dumps(line), flush=True)
        del layer, io
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
