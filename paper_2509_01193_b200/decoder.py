"""One Llama decoder layer's fine-tuning step over a packed multi-task batch.

The unit the paper's cost model profiles (App. D: "we simplify and expedite the
offline process by profiling only a single layer"; attention ~ s^2, other modules ~ s).
Public Llama-2 layer (reading Q27; oracle/decoder.py is its fp64 definition):

    h1 = RMSNorm(X) g_attn;  q, k, v = LoRA projections of h1;  q, k = RoPE (per sequence)
    a  = causal attention inside every packed sequence;  o = LoRA projection of a
    x2 = X + o;  h2 = RMSNorm(x2) g_mlp;  gate, up = LoRA projections of h2
    Y  = x2 + down(silu(gate) * up)

Our kernels (C ABI, liblobra.so): the seven LoRA projections (q/k/v and gate/up as
projection groups), RMSNorm with the fused residual add / residual-gradient add, RoPE,
SwiGLU, the last residual add.  Attention (attention.py): cuDNN's ragged SDPA by default (a
library call like cuBLAS; faster than ours today), `attn_backend="lobra"` for our own tcgen05
forward and backward (csrc/attn.cu), FlashAttention-2 varlen as a further
alternative.  PyTorch only allocates memory.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .attention import make_attention
from .layer import LLAMA2_7B, LoraLayer


class DecoderLayer:
    def __init__(self, shapes=LLAMA2_7B, n_heads=32, ranks=(16,), scales=(2.0,), device="cuda:0",
                 dtype=torch.bfloat16, seed=0, eps=1e-5, theta=10000.0, group_inputs=True,
                 deterministic_attn=False, attn_backend="cudnn"):
        assert dtype == torch.bfloat16, "the decoder layer runs the bf16 path"
        self.dev = torch.device(device)
        self.lora = LoraLayer(shapes, ranks, scales, self.dev, dtype, seed=seed, group_inputs=group_inputs)
        self.h = next(p.d_in for p in self.lora.projs if p.name == "q")
        self.f = next(p.d_out for p in self.lora.projs if p.name == "gate")
        self.n_heads = n_heads
        self.head_dim = self.h // n_heads
        self.hk = next(p.d_out for p in self.lora.projs if p.name == "k")    # kv width
        self.n_kv_heads = self.hk // self.head_dim      # < n_heads: grouped-query attention (70B)
        self.eps, self.theta = eps, theta
        self.attn = make_attention(attn_backend, n_heads, self.head_dim, self.dev, deterministic_attn,
                                   self.n_kv_heads)
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed + 7)
        # frozen RMSNorm gains (synthetic: 1 + N(0, 0.1^2))
        self.g_attn = (1 + 0.1 * torch.randn(self.h, generator=g, device=self.dev)).to(dtype)
        self.g_mlp = (1 + 0.1 * torch.randn(self.h, generator=g, device=self.dev)).to(dtype)
        self.cache = {}
        self.saved = None
        self._ctx, self._ctxs = 0, {}

    # ------------------------------------------------------------------ micro-batch contexts
    def select_context(self, k):
        """Pipeline schedules (1F1B, pipeline.py) keep several micro-batches in flight: each
        context k owns its activations (the buffer cache and the saved state of forward) and
        the projections' saved H_s; the adapter gradients and workspaces are shared."""
        if k == self._ctx:
            return
        L = self.lora
        self._ctxs[self._ctx] = (self.cache, self.saved, L.group_Hs, [p.Hs for p in L.projs])
        c = self._ctxs.pop(k, None)
        if c is None:
            self.cache, self.saved, L.group_Hs = {}, None, {}
            for p in L.projs:
                p.Hs = None
        else:
            self.cache, self.saved, L.group_Hs, hs = c
            for p, h in zip(L.projs, hs):
                p.Hs = h
        self._ctx = k

    # ------------------------------------------------------------------ buffers
    def _buf(self, name, shape, dtype=torch.bfloat16):
        t = self.cache.get(name)
        n = int(np.prod(shape))
        if t is None or t.numel() < n or t.dtype != dtype:
            t = torch.empty(n, device=self.dev, dtype=dtype)
            self.cache[name] = t
        return t[:n].view(*shape)

    # ------------------------------------------------------------------ forward
    def forward(self, seq_lens, seq_task, X, stream=None):
        """X [T, h] bf16 (device) -> Y [T, h]; keeps the activations for backward()."""
        seq_lens = np.asarray(seq_lens, np.int32)
        seq_task = np.asarray(seq_task, np.int32)
        T, h, f, hk = int(seq_lens.sum()), self.h, self.f, self.hk
        H, D, Hk = self.n_heads, self.head_dim, self.n_kv_heads
        L = self.lora
        L.ensure(seq_lens, seq_task)
        cu = torch.from_numpy(np.concatenate([[0], np.cumsum(seq_lens)]).astype(np.int32)).to(self.dev)
        maxlen = int(seq_lens.max()) if len(seq_lens) else 0
        b = self._buf
        h1, x2, h2 = b("h1", (T, h)), b("x2", (T, h)), b("h2", (T, h))
        q, k, v, o = b("q", (T, h)), b("k", (T, hk)), b("v", (T, hk)), b("o", (T, h))
        gate, up, act, down = b("gate", (T, f)), b("up", (T, f)), b("act", (T, f)), b("down", (T, h))
        r1, r2 = b("r1", (T,), torch.float32), b("r2", (T,), torch.float32)
        Y = b("Y", (T, h))
        _lib.lobra_rmsnorm_fwd(X, self.g_attn, self.eps, h1, r1, stream=stream)
        L.forward_group("attn", seq_lens, seq_task, h1, {"q": q, "k": k, "v": v}, stream)
        if Hk == H:
            _lib.lobra_rope(cu, T, H, D, self.theta, q, k, stream=stream)
        else:
            _lib.lobra_rope(cu, T, H, D, self.theta, q, stream=stream)
            _lib.lobra_rope(cu, T, Hk, D, self.theta, k, stream=stream)
        att, lse, actx = self.attn.forward(q.view(T, H, D), k.view(T, Hk, D), v.view(T, Hk, D), seq_lens)
        L.forward_group("o_in", seq_lens, seq_task, att.view(T, h), {"o": o}, stream)
        _lib.lobra_rmsnorm_fwd(X, self.g_mlp, self.eps, h2, r2, R=o, S_out=x2, stream=stream)
        L.forward_group("mlp", seq_lens, seq_task, h2, {"gate": gate, "up": up}, stream)
        _lib.lobra_swiglu_fwd(gate, up, act, stream=stream)
        L.forward_group("down_in", seq_lens, seq_task, act, {"down": down}, stream)
        _lib.lobra_add(x2, down, Y, stream=stream)
        self.saved = dict(seq_lens=seq_lens, seq_task=seq_task, cu=cu, maxlen=maxlen, X=X, att=att, lse=lse, T=T,
                          actx=actx)
        return Y

    # ------------------------------------------------------------------ backward
    def backward(self, dY, accumulate_dadb=False, stream=None):
        """dY [T, h] -> dX [T, h]; adapter gradients (+)= into self.lora.flat_grad."""
        s = self.saved
        seq_lens, seq_task, cu, maxlen, T = s["seq_lens"], s["seq_task"], s["cu"], s["maxlen"], s["T"]
        h, f, H, D, hk, Hk = self.h, self.f, self.n_heads, self.head_dim, self.hk, self.n_kv_heads
        L = self.lora
        b = self._buf
        c = self.cache
        d_act, d_gate, d_up = b("d_act", (T, f)), b("d_gate", (T, f)), b("d_up", (T, f))
        dh2, dx2, d_att, dh1 = b("dh2", (T, h)), b("dx2", (T, h)), b("d_att", (T, h)), b("dh1", (T, h))
        dq, dk, dv = b("dq", (T, h)), b("dk", (T, hk)), b("dv", (T, hk))
        dX = b("dX", (T, h))
        q, k, v = c["q"][:T * h].view(T, h), c["k"][:T * hk].view(T, hk), c["v"][:T * hk].view(T, hk)
        gate, up = c["gate"][:T * f].view(T, f), c["up"][:T * f].view(T, f)
        act, h2, x2, h1 = (c[n][:T * w].view(T, w) for n, w in (("act", f), ("h2", h), ("x2", h), ("h1", h)))
        L.backward_group("down_in", seq_lens, seq_task, act, {"down": dY}, d_act, accumulate_dadb, stream)
        _lib.lobra_swiglu_bwd(d_act, gate, up, d_gate, d_up, stream=stream)
        L.backward_group("mlp", seq_lens, seq_task, h2, {"gate": d_gate, "up": d_up}, dh2, accumulate_dadb, stream)
        _lib.lobra_rmsnorm_bwd(dh2, x2, self.g_mlp, c["r2"][:T], dx2, dRes=dY, stream=stream)
        L.backward_group("o_in", seq_lens, seq_task, s["att"].view(T, h), {"o": dx2}, d_att, accumulate_dadb, stream)
        self.attn.backward(d_att.view(T, H, D), q.view(T, H, D), k.view(T, Hk, D), v.view(T, Hk, D), s["att"],
                           s["lse"], s["actx"], dq.view(T, H, D), dk.view(T, Hk, D), dv.view(T, Hk, D))
        if Hk == H:
            _lib.lobra_rope(cu, T, H, D, self.theta, dq, dk, inverse=True, stream=stream)
        else:
            _lib.lobra_rope(cu, T, H, D, self.theta, dq, inverse=True, stream=stream)
            _lib.lobra_rope(cu, T, Hk, D, self.theta, dk, inverse=True, stream=stream)
        L.backward_group("attn", seq_lens, seq_task, h1, {"q": dq, "k": dk, "v": dv}, dh1, accumulate_dadb, stream)
        _lib.lobra_rmsnorm_bwd(dh1, s["X"], self.g_attn, c["r1"][:T], dX, dRes=dx2, stream=stream)
        return dX

    def flops(self, seq_lens) -> dict:
        """Algorithmic FLOPs of fwd + bwd (frozen base: no dW): projections 4 T sum(in out)
        + LoRA 6 T r sum(in + out); causal attention fwd 2 * 2 sum_s s^2/2 h (QK^T, PV) and
        bwd 2.5x that (dQ, dK, dV, dS recompute: 5 matmuls of the same size)."""
        T = int(np.sum(seq_lens))
        proj = 4 * T * sum(p.d_in * p.d_out for p in self.lora.projs)
        r = float(np.mean(self.lora.ranks))
        lora = 6 * T * r * sum(p.d_in + p.d_out for p in self.lora.projs)
        s2 = float(np.sum(np.asarray(seq_lens, np.float64) ** 2)) / 2
        att_f = 4 * s2 * self.h          # per query head (GQA shares k, v but not the matmuls)
        return {"proj": proj, "lora": lora, "attn": att_f * 3.5, "total": proj + lora + att_f * 3.5}
