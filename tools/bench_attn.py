"""Attention forward and backward (varlen causal, D = 128) device time: own tcgen05 kernels vs
cuDNN ragged SDPA vs FlashAttention-2 (run under gpurun).  Causal FLOPs: forward
2 * 2 * sum(L^2)/2 * H * D, backward 2.5x that (five matmuls of the same size)."""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_01193_b200.attention import make_attention  # noqa: E402
from workloads import synth  # noqa: E402


def timeit(fn, n=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    out = {}
    cases = {"c2_T16384_H32": (synth.config_c2().seq_lens.tolist(), 32, 32),
             "long_4seq_H32": ([4096, 2048, 6000, 4240], 32, 32),
             "gqa70b_H64_kv8": (synth.config_c2().seq_lens.tolist(), 64, 8)}
    for name, (lens, H, Hkv) in cases.items():
        lens = [int(x) for x in lens if x > 0]
        T = sum(lens)
        g = torch.Generator(device="cuda").manual_seed(0)
        q = torch.randn(T, H, 128, generator=g, device="cuda").to(torch.bfloat16)
        k = torch.randn(T, Hkv, 128, generator=g, device="cuda").to(torch.bfloat16)
        v = torch.randn(T, Hkv, 128, generator=g, device="cuda").to(torch.bfloat16)
        flops = 2.0 * sum(l * l for l in lens) * H * 128
        res = {}
        for be in ("lobra", "cudnn", "flash_attn"):
            a = make_attention(be, H, 128, "cuda", n_kv_heads=Hkv)
            ln = np.array(lens, np.int32)
            ms = timeit(lambda: a.forward(q, k, v, ln))
            o, lse, ctx = a.forward(q, k, v, ln)
            dO = torch.randn(T, H, 128, generator=g, device="cuda").to(torch.bfloat16)
            dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
            msb = timeit(lambda: a.backward(dO, q, k, v, o, lse, ctx, dq, dk, dv))
            res[be] = {"ms": ms, "TFLOPs": flops / ms / 1e9, "bwd_ms": msb, "bwd_TFLOPs": 2.5 * flops / msb / 1e9}
        out[name] = res
        print(name, json.dumps(res), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
