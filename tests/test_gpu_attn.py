"""GPU: the own tcgen05 varlen causal attention forward (csrc/attn.cu) against
the fp64 oracle attention (oracle/decoder.py, pinned to HF Llama) on the same bf16 inputs,
and against FlashAttention-2's forward; grouped-query heads, ragged sequences (1 token,
lengths not multiples of 128, several 128-tiles).  Tolerance: O is rounded to bf16 once and
P is rounded to bf16 before P V (as in FlashAttention): 1e-2 (max-norm relative); LSE
absolute 1e-3 (fp32 arithmetic)."""
import math

import numpy as np
import pytest

from oracle import decoder as Dd
from oracle import lora as O

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("lens,H,Hkv", [([1, 300, 57, 129, 200, 33], 4, 2), ([128, 256, 384], 2, 2),
                                        ([1000, 17, 520], 4, 1)])
def test_attn_fwd_matches_oracle(lens, H, Hkv):
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    T = sum(lens)
    g = torch.Generator(device="cuda")
    g.manual_seed(T + H)
    q = torch.randn(T, H, 128, generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn(T, Hkv, 128, generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn(T, Hkv, 128, generator=g, device="cuda").to(torch.bfloat16)
    o = torch.full_like(q, float("nan"))
    lse = torch.full((H, T), float("nan"), device="cuda")
    ws = torch.empty(_lib.lobra_attn_workspace_bytes(lens, H), dtype=torch.uint8, device="cuda")
    _lib.lobra_attn_fwd(lens, q, k, v, o, lse, ws)
    torch.cuda.synchronize()
    f = lambda x: x.float().cpu().numpy().astype(np.float64)
    ao, Ps = Dd.attention(f(q), f(k), f(v), lens)
    assert O.max_rel_err(f(o), ao) <= 1e-2
    # LSE from the oracle's logits: log sum_k exp(q k / sqrt(D)) over the causal prefix
    qo, ko = f(q), np.repeat(f(k), H // Hkv, axis=1)
    ref = np.zeros((H, T))
    off = 0
    for n in lens:
        for h in range(H):
            S = qo[off:off + n, h] @ ko[off:off + n, h].T / math.sqrt(128)
            S = np.where(np.tril(np.ones((n, n), bool)), S, -np.inf)
            mx = S.max(axis=1, keepdims=True)
            ref[h, off:off + n] = (mx + np.log(np.exp(S - mx).sum(axis=1, keepdims=True)))[:, 0]
        off += n
    assert np.max(np.abs(lse.cpu().numpy() - ref)) <= 1e-3


def test_attn_fwd_agrees_with_flash_attention():
    torch = _torch()
    fa = pytest.importorskip("flash_attn.flash_attn_interface")
    from paper_2509_01193_b200 import _lib
    lens = [4096, 1500, 33, 2700]
    T, H = sum(lens), 8
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    q, k, v = (torch.randn(T, H, 128, generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    lse = torch.empty(H, T, device="cuda")
    ws = torch.empty(_lib.lobra_attn_workspace_bytes(lens, H), dtype=torch.uint8, device="cuda")
    _lib.lobra_attn_fwd(lens, q, k, v, o, lse, ws)
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    o2, lse2, _, _ = fa._flash_attn_varlen_forward(q, k, v, cu, cu, max(lens), max(lens), 0.0, 1 / math.sqrt(128), True)
    torch.cuda.synchronize()
    f = lambda x: x.float().cpu().numpy().astype(np.float64)
    assert O.max_rel_err(f(o), f(o2)) <= 1e-2
    assert float((lse - lse2).abs().max()) <= 1e-3


# ------------------------------------------------------------------ backward (lobra_attn_bwd)
# P and dS are rounded to bf16 before the tcgen05 products (as FlashAttention does), dQ/dK/dV
# once more on output; the north-star bf16 tolerance 2e-2 (max-norm relative, per tensor).
def _attn_bwd_case(torch, lens, H, Hkv, seed):
    from paper_2509_01193_b200 import _lib
    T = sum(lens)
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    q = torch.randn(T, H, 128, generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn(T, Hkv, 128, generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn(T, Hkv, 128, generator=g, device="cuda").to(torch.bfloat16)
    dO = torch.randn(T, H, 128, generator=g, device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    lse = torch.empty(H, T, device="cuda")
    ws = torch.empty(_lib.lobra_attn_workspace_bytes(lens, H), dtype=torch.uint8, device="cuda")
    _lib.lobra_attn_fwd(lens, q, k, v, o, lse, ws)
    dq = torch.full_like(q, float("nan"))
    dk = torch.full_like(k, float("nan"))
    dv = torch.full_like(v, float("nan"))
    wsb = torch.empty(_lib.lobra_attn_bwd_workspace_bytes(lens, H, Hkv), dtype=torch.uint8, device="cuda")
    _lib.lobra_attn_bwd(lens, q, k, v, o, dO, lse, dq, dk, dv, wsb)
    torch.cuda.synchronize()
    return q, k, v, o, dO, lse, dq, dk, dv


@pytest.mark.parametrize("lens,H,Hkv", [([1, 300, 57, 129, 200, 33], 4, 2), ([128, 256, 384], 2, 2),
                                        ([1000, 17, 520], 4, 1), ([5], 1, 1)])
def test_attn_bwd_matches_oracle(lens, H, Hkv):
    torch = _torch()
    q, k, v, o, dO, lse, dq, dk, dv = _attn_bwd_case(torch, lens, H, Hkv, seed=sum(lens) * 3 + H)
    f = lambda x: x.float().cpu().numpy().astype(np.float64)
    _, Ps = Dd.attention(f(q), f(k), f(v), lens)
    rq, rk, rv = Dd.attention_bwd(f(dO), f(q), f(k), f(v), Ps, lens)
    errs = {"dq": O.max_rel_err(f(dq), rq), "dk": O.max_rel_err(f(dk), rk), "dv": O.max_rel_err(f(dv), rv)}
    assert all(e <= 2e-2 for e in errs.values()), errs


def test_attn_bwd_agrees_with_flash_attention():
    torch = _torch()
    fa = pytest.importorskip("flash_attn.flash_attn_interface")
    lens = [4096, 1500, 33, 2700]
    H = 8
    q, k, v, o, dO, lse, dq, dk, dv = _attn_bwd_case(torch, lens, H, H, seed=11)
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    dq2, dk2, dv2 = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    fa._flash_attn_varlen_backward(dO, q, k, v, o, lse, dq2, dk2, dv2, cu, cu, max(lens), max(lens), 0.0,
                                   1 / math.sqrt(128), True, -1, -1, 0.0, None, True)
    torch.cuda.synchronize()
    f = lambda x: x.float().cpu().numpy().astype(np.float64)
    errs = {"dq": O.max_rel_err(f(dq), f(dq2)), "dk": O.max_rel_err(f(dk), f(dk2)),
            "dv": O.max_rel_err(f(dv), f(dv2))}
    assert all(e <= 2e-2 for e in errs.values()), errs
