"""Decoder-layer benchmark and App. D cost-model fit (run under gpurun).

    python tools/bench_layer.py [--steps 10] [--fit] [--out profiles/r1_layer_cost.json]

1. One Llama-2-7B decoder layer (paper_2509_01193_b200/decoder.py: our LoRA projection
   groups, RMSNorm / RoPE / SwiGLU kernels, library varlen attention) fwd + bwd on the C2
   workload (T = 16384 packed tokens, 4 tasks r = 16, lengths <= 4096): tokens/s, device
   time per class (our kernels from the library's CUDA events; attention + glue = rest).
2. --fit: the paper's per-layer cost model (App. D: t(b, s) proportional to b,
   quadratic in s; profiled on a single layer) measured on chunks of b sequences of
   length s and fitted by least squares as t = c0 + c1 * b s + c2 * b s^2 (reading Q28:
   c0 = per-chunk fixed cost, which the paper's t(b, s) folds into b); leave-one-out
   prediction error reported (the paper's cost model is "within 10%", §5.3).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed_layer(layer, lens, tasks, X, dY, reps, warm=2):
    import torch
    from paper_2509_01193_b200 import _lib
    for _ in range(warm):
        layer.forward(lens, tasks, X)
        layer.backward(dY)
    torch.cuda.synchronize()
    _lib.lobra_profile_enable(True)
    _lib.lobra_profile_read(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        layer.forward(lens, tasks, X)
        layer.backward(dY)
    e1.record()
    torch.cuda.synchronize()
    prof = _lib.lobra_profile_read(reset=True)
    _lib.lobra_profile_enable(False)
    ms = e0.elapsed_time(e1) / reps
    return ms, {k: v[1] / reps for k, v in prof.items() if v[0]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--fit", action="store_true")
    ap.add_argument("--attn", default="cudnn", choices=["cudnn", "flash_attn", "lobra"])
    ap.add_argument("--model", default="7b", choices=["7b", "70b"])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_layer_cost.json"))
    args = ap.parse_args()
    import torch
    from paper_2509_01193_b200.decoder import DecoderLayer
    from paper_2509_01193_b200.layer import LLAMA2_7B, LLAMA2_70B
    from workloads import synth

    torch.cuda.set_device(0)
    tasks = synth.c2_tasks()
    ranks, scales = [t.rank for t in tasks], [t.scale for t in tasks]
    shapes, heads, hid = (LLAMA2_7B, 32, 4096) if args.model == "7b" else (LLAMA2_70B, 64, 8192)
    layer = DecoderLayer(shapes, n_heads=heads, ranks=ranks, scales=scales, seed=11, attn_backend=args.attn)
    Tmax = 16384
    g = torch.Generator(device="cuda")
    g.manual_seed(12)
    Xb = torch.randn(Tmax, hid, generator=g, device="cuda").to(torch.bfloat16)
    dYb = torch.randn(Tmax, hid, generator=g, device="cuda").to(torch.bfloat16)

    wl = synth.config_c2()
    T = wl.T
    ms, cls = timed_layer(layer, wl.seq_lens, wl.seq_task, Xb[:T], dYb[:T], args.steps)
    fl = layer.flops(wl.seq_lens)
    ours = sum(cls.values())
    line = {"metric": f"Llama-2-{args.model.upper()} decoder layer fwd+bwd tokens/s (NEXT-3, 1 GPU)",
            "value": T / (ms / 1e3),
            "unit": "tokens/s", "ms_per_step": ms, "steps": args.steps, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "C2 (T=16384, 4 tasks r=16, lengths <= 4096)", "layer": f"llama2-{args.model}" + (" (GQA 64/8 heads, TP1)" if args.model == "70b" else ""),
                       "attention": {"cudnn": "cuDNN 9 ragged SDPA (library)",
                                     "flash_attn": "flash_attn 2.8 varlen (library)",
                                     "lobra": "own tcgen05 forward + backward (csrc/attn.cu)"}[args.attn]},
            "algorithmic_tflops": fl["total"] / (ms / 1e3) / 1e12,
            "flops_share": {k: fl[k] / fl["total"] for k in ("proj", "lora", "attn")},
            "ms_by_class": cls, "ms_attention_and_glue": ms - ours}
    print(json.dumps(line), flush=True)
    if not args.fit:
        return
    # ---- App. D cost model: chunks of b sequences of length s (one task each, round robin)
    pts = []
    for s in (256, 512, 1024, 2048, 4096, 8192):
        for total in (4096, 8192, 16384):
            b = total // s
            if b < 1:
                continue
            lens = np.full(b, s, np.int32)
            tids = (np.arange(b) % len(ranks)).astype(np.int32)
            o = np.argsort(tids, kind="stable")
            lens, tids = lens[o], tids[o]
            t_ms, _ = timed_layer(layer, lens, tids, Xb[:b * s], dYb[:b * s], max(3, args.steps // 2), warm=1)
            pts.append({"b": int(b), "s": int(s), "ms": t_ms})
            print(json.dumps(pts[-1]), flush=True)
    A = np.array([[1.0, p["b"] * p["s"], p["b"] * p["s"] ** 2] for p in pts])
    y = np.array([p["ms"] for p in pts])
    coef, *_ = np.linalg.lstsq(A, y, rcond=None)
    loo = []
    for i in range(len(pts)):
        m = np.arange(len(pts)) != i
        c, *_ = np.linalg.lstsq(A[m], y[m], rcond=None)
        loo.append(abs(A[i] @ c - y[i]) / y[i])
    res = {"model": f"t_ms = c0 + c1 * b s + c2 * b s^2 (App. D P:1485, one {args.model} layer fwd+bwd, 1 B200)",
           "attention": args.attn,
           "c0_ms": coef[0], "c1_ms_per_token": coef[1], "c2_ms_per_token_len": coef[2],
           "points": pts, "fit_rel_err": [abs(A[i] @ coef - y[i]) / y[i] for i in range(len(pts))],
           "loo_rel_err_max": max(loo), "loo_rel_err_mean": float(np.mean(loo)), "c2_layer_line": line,
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)
    print(json.dumps({k: res[k] for k in ("c0_ms", "c1_ms_per_token", "c2_ms_per_token_len", "loo_rel_err_max",
                                          "loo_rel_err_mean")}))


if __name__ == "__main__":
    main()
