"""Probe: which attention libraries in the image run varlen causal attention on this GPU."""
import time
import torch

dev = torch.device("cuda:0")
print(torch.cuda.get_device_name(0), torch.cuda.get_device_capability(0))
T, H, D = 16384, 32, 128
lens = [4096, 2048, 6000, 4240]
cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), dtype=torch.int32, device=dev)
q = torch.randn(T, H, D, device=dev, dtype=torch.bfloat16)
k = torch.randn(T, H, D, device=dev, dtype=torch.bfloat16)
v = torch.randn(T, H, D, device=dev, dtype=torch.bfloat16)


def bench(fn, n=10):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3


try:
    import flash_attn
    from flash_attn import flash_attn_varlen_func
    print("flash_attn", flash_attn.__version__)
    f = lambda: flash_attn_varlen_func(q, k, v, cu, cu, max(lens), max(lens), causal=True)
    print("fa2 fwd ms", bench(f))
    qq, kk, vv = (x.clone().requires_grad_() for x in (q, k, v))
    o = flash_attn_varlen_func(qq, kk, vv, cu, cu, max(lens), max(lens), causal=True)
    g = torch.randn_like(o)
    print("fa2 bwd ms", bench(lambda: torch.autograd.grad(flash_attn_varlen_func(qq, kk, vv, cu, cu, max(lens), max(lens), causal=True), (qq, kk, vv), g)))
except Exception as e:
    print("flash_attn failed:", repr(e)[:300])
try:
    import flashinfer
    print("flashinfer", flashinfer.__version__)
except Exception as e:
    print("flashinfer failed:", repr(e)[:300])
try:
    from torch.nn.attention.varlen import varlen_attn
    print("torch varlen_attn available")
except Exception as e:
    print("torch varlen:", repr(e)[:200])
try:
    import torch.nn.functional as F
    qb = q[:4096].transpose(0, 1).unsqueeze(0)
    print("sdpa 4096 causal ms", bench(lambda: F.scaled_dot_product_attention(qb, qb, qb, is_causal=True)))
except Exception as e:
    print("sdpa failed", repr(e)[:200])
