"""Probe: fwd+bwd time of varlen causal attention backends on this GPU (T = 16384)."""
import time
import torch
import torch.nn.functional as F

dev = torch.device("cuda:0")
T, H, D = 16384, 32, 128
lens = [4096, 2048, 6000, 4240]
cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), dtype=torch.int32, device=dev)


def bench(fn, n=10):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3


q, k, v = (torch.randn(T, H, D, device=dev, dtype=torch.bfloat16, requires_grad=True) for _ in range(3))
g = torch.randn(T, H, D, device=dev, dtype=torch.bfloat16)
flops = 2 * H * D * sum(l * l for l in lens)   # causal fwd (QK^T + PV, half of s^2 each)
try:
    from torch.nn.attention.varlen import varlen_attn
    import inspect
    print(inspect.signature(varlen_attn))
    f = lambda: varlen_attn(q, k, v, cu, cu, max(lens), max(lens), is_causal=True)
    ms = bench(f)
    print("torch varlen fwd ms", ms, "TF/s", flops / ms / 1e9)
    fb = lambda: torch.autograd.grad(varlen_attn(q, k, v, cu, cu, max(lens), max(lens), is_causal=True), (q, k, v), g)
    ms = bench(fb)
    print("torch varlen fwd+bwd ms", ms, "TF/s", 3.5 * flops / ms / 1e9)
except Exception as e:
    print("torch varlen failed", repr(e)[:300])
from flash_attn import flash_attn_varlen_func
ms = bench(lambda: torch.autograd.grad(flash_attn_varlen_func(q, k, v, cu, cu, max(lens), max(lens), causal=True), (q, k, v), g))
print("fa2 fwd+bwd ms", ms, "TF/s", 3.5 * flops / ms / 1e9)
# cuDNN SDPA per sequence (padded batch of 1 per sequence)
from torch.nn.attention import sdpa_kernel, SDPBackend
for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION):
    try:
        qs = [q[cu[i]:cu[i + 1]].transpose(0, 1)[None].detach().requires_grad_() for i in range(len(lens))]
        def run():
            outs = []
            with sdpa_kernel(be):
                for x in qs:
                    o = F.scaled_dot_product_attention(x, x, x, is_causal=True)
                    outs.append(o)
            torch.autograd.grad(outs, qs, [torch.ones_like(o) for o in outs])
        ms = bench(run)
        print(be, "per-seq fwd+bwd ms", ms, "TF/s", 3.5 * flops / ms / 1e9)
    except Exception as e:
        print(be, "failed", repr(e)[:200])
