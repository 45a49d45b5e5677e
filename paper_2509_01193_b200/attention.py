"""Varlen causal attention for the decoder layer.

Attention is not on the north-star path; three backends over the packed layout q, k, v
[T, H, D] with per-sequence causal masks (block-diagonal over the pack):

  * "cudnn" (default): cuDNN 9 frontend SDPA forward / backward on RAGGED tensors (THD
    layout: the sequences of the pack addressed through ragged offsets, no padding copies);
    graphs are built once per (batch bucket, max-length bucket) and cached -- a library
    call like cuBLAS, and today the fastest;
  * "lobra": our own tcgen05 kernels, forward (lobra_attn_fwd) and backward
    (lobra_attn_bwd, recomputation from the forward's LSE), csrc/attn.cu;
  * "flash_attn": FlashAttention-2 varlen kernels (mma.sync; ~3x slower on B200).
"""
from __future__ import annotations

import math

import numpy as np
import torch


def _bucket(x: int, q: int) -> int:
    return max(q, (x + q - 1) // q * q)


class CudnnVarlenAttention:
    def __init__(self, n_heads: int, head_dim: int, device, n_kv_heads: int | None = None):
        import cudnn
        self.cudnn = cudnn
        self.H, self.D = n_heads, head_dim
        self.Hkv = n_kv_heads or n_heads      # grouped-query attention when < n_heads
        self.dev = torch.device(device)
        self.handle = cudnn.create_handle()
        self.graphs = {}
        self.ws = torch.empty(0, dtype=torch.uint8, device=self.dev)

    # -------------------------------------------------------------- graph construction
    def _graph(self, kind: str, B: int, S: int):
        key = (kind, B, S)
        if key in self.graphs:
            return self.graphs[key]
        c = self.cudnn
        H, Hk, D = self.H, self.Hkv, self.D
        g = c.pygraph(io_data_type=c.data_type.BFLOAT16, intermediate_data_type=c.data_type.FLOAT,
                      compute_data_type=c.data_type.FLOAT, handle=self.handle)
        dim, stride = [B, H, S, D], [S * H * D, D, H * D, 1]
        dimk, stridek = [B, Hk, S, D], [S * Hk * D, D, Hk * D, 1]

        def ragged(name, kv=False):
            off = g.tensor(name=name + "_off", dim=[B + 1, 1, 1, 1], stride=[1, 1, 1, 1],
                           data_type=c.data_type.INT32)
            return g.tensor(name=name, dim=dimk if kv else dim, stride=stridek if kv else stride,
                            data_type=c.data_type.BFLOAT16, ragged_offset=off), off

        t = {}
        t["q"], t["q_off"] = ragged("q")
        t["k"], t["k_off"] = ragged("k", True)
        t["v"], t["v_off"] = ragged("v", True)
        t["sq"] = g.tensor(name="seq_q", dim=[B, 1, 1, 1], stride=[1, 1, 1, 1], data_type=c.data_type.INT32)
        t["skv"] = g.tensor(name="seq_kv", dim=[B, 1, 1, 1], stride=[1, 1, 1, 1], data_type=c.data_type.INT32)
        scale = 1.0 / math.sqrt(D)
        if kind == "fwd":
            o, stats = g.sdpa(name="sdpa", q=t["q"], k=t["k"], v=t["v"], is_inference=False, attn_scale=scale,
                              use_causal_mask=True, use_padding_mask=True, seq_len_q=t["sq"], seq_len_kv=t["skv"])
            t["o_off"] = g.tensor(name="o_off", dim=[B + 1, 1, 1, 1], stride=[1, 1, 1, 1], data_type=c.data_type.INT32)
            o.set_output(True).set_dim(dim).set_stride(stride).set_ragged_offset(t["o_off"])
            stats.set_output(True).set_data_type(c.data_type.FLOAT).set_dim([B, H, S, 1]).set_stride(
                [H * S, S, 1, 1])
            t["o"], t["stats"] = o, stats
        else:
            t["o"], t["o_off"] = ragged("o")
            t["dO"], t["dO_off"] = ragged("dO")
            t["stats"] = g.tensor(name="stats", dim=[B, H, S, 1], stride=[H * S, S, 1, 1],
                                  data_type=c.data_type.FLOAT)
            dq, dk, dv = g.sdpa_backward(name="sdpa_bwd", q=t["q"], k=t["k"], v=t["v"], o=t["o"], dO=t["dO"],
                                         stats=t["stats"], attn_scale=scale, use_causal_mask=True,
                                         use_padding_mask=True, seq_len_q=t["sq"], seq_len_kv=t["skv"])
            for n, x in (("dq", dq), ("dk", dk), ("dv", dv)):
                t[n + "_off"] = g.tensor(name=n + "_off", dim=[B + 1, 1, 1, 1], stride=[1, 1, 1, 1],
                                         data_type=c.data_type.INT32)
                kv = n != "dq"
                x.set_output(True).set_dim(dimk if kv else dim).set_stride(stridek if kv else stride) \
                    .set_ragged_offset(t[n + "_off"])
                t[n] = x
        g.validate()
        g.build_operation_graph()
        g.create_execution_plans([c.heur_mode.A, c.heur_mode.FALLBACK])
        g.check_support()
        g.build_plans()
        self.graphs[key] = (g, t)
        return g, t

    def _meta(self, seq_lens):
        """Batch / length buckets and the device int32 tensors (offsets in elements)."""
        n = len(seq_lens)
        B = _bucket(n, 8)
        S = _bucket(int(max(seq_lens)) if n else 1, 128)
        lens = np.zeros(B, np.int32)
        lens[:n] = seq_lens
        cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        off = torch.from_numpy((cu * self.H * self.D).astype(np.int32)).to(self.dev).view(B + 1, 1, 1, 1)
        offk = torch.from_numpy((cu * self.Hkv * self.D).astype(np.int32)).to(self.dev).view(B + 1, 1, 1, 1)
        sl = torch.from_numpy(lens).to(self.dev).view(B, 1, 1, 1)
        return B, S, (off, offk), sl

    def _run(self, g, pack):
        need = g.get_workspace_size()
        if self.ws.numel() < need:
            self.ws = torch.empty(need, dtype=torch.uint8, device=self.dev)
        self.cudnn.set_stream(handle=self.handle, stream=torch.cuda.current_stream().cuda_stream)
        g.execute(pack, self.ws, handle=self.handle)

    # -------------------------------------------------------------- public
    def forward(self, q, k, v, seq_lens):
        """q, k, v [T, H, D] bf16 -> (o [T, H, D], stats [B, H, S, 1] fp32, ctx)."""
        B, S, (off, offk), sl = self._meta(seq_lens)
        g, t = self._graph("fwd", B, S)
        o = torch.empty_like(q)
        stats = torch.empty(B, self.H, S, 1, dtype=torch.float32, device=self.dev)
        self._run(g, {t["q"]: q, t["k"]: k, t["v"]: v, t["o"]: o, t["stats"]: stats, t["q_off"]: off,
                      t["k_off"]: offk, t["v_off"]: offk, t["o_off"]: off, t["sq"]: sl, t["skv"]: sl})
        return o, stats, (B, S, (off, offk), sl)

    def backward(self, dO, q, k, v, o, stats, ctx, dq, dk, dv):
        B, S, (off, offk), sl = ctx
        g, t = self._graph("bwd", B, S)
        self._run(g, {t["q"]: q, t["k"]: k, t["v"]: v, t["o"]: o, t["dO"]: dO, t["stats"]: stats,
                      t["dq"]: dq, t["dk"]: dk, t["dv"]: dv, t["q_off"]: off, t["k_off"]: offk, t["v_off"]: offk,
                      t["o_off"]: off, t["dO_off"]: off, t["dq_off"]: off, t["dk_off"]: offk, t["dv_off"]: offk,
                      t["sq"]: sl, t["skv"]: sl})


class FlashVarlenAttention:
    """FlashAttention-2 varlen kernels (library, mma.sync)."""

    def __init__(self, n_heads: int, head_dim: int, device, deterministic=False):
        from flash_attn import flash_attn_interface as fa
        self.fa, self.D, self.det = fa, head_dim, deterministic
        self.dev = torch.device(device)

    def forward(self, q, k, v, seq_lens):
        cu = torch.from_numpy(np.concatenate([[0], np.cumsum(seq_lens)]).astype(np.int32)).to(self.dev)
        m = int(max(seq_lens)) if len(seq_lens) else 0
        o, lse, _, _ = self.fa._flash_attn_varlen_forward(q, k, v, cu, cu, m, m, 0.0, 1.0 / math.sqrt(self.D), True)
        return o, lse, (cu, m)

    def backward(self, dO, q, k, v, o, lse, ctx, dq, dk, dv):
        cu, m = ctx
        self.fa._flash_attn_varlen_backward(dO, q, k, v, o, lse, dq, dk, dv, cu, cu, m, m, 0.0,
                                            1.0 / math.sqrt(self.D), True, -1, -1, 0.0, None, self.det)


class LobraVarlenAttention:
    """Own tcgen05 kernels for both directions: lobra_attn_fwd (O, LSE [H, T]) and
    lobra_attn_bwd (recomputation from the LSE; csrc/attn.cu)."""

    def __init__(self, n_heads: int, head_dim: int, device, n_kv_heads: int | None = None):
        from . import _lib
        self.lib, self.H, self.D = _lib, n_heads, head_dim
        self.Hkv = n_kv_heads or n_heads
        self.dev = torch.device(device)
        self.ws = torch.empty(0, dtype=torch.uint8, device=self.dev)

    def _ws(self, need):
        if self.ws.numel() < need:
            self.ws = torch.empty(need, dtype=torch.uint8, device=self.dev)
        return self.ws

    def forward(self, q, k, v, seq_lens):
        lens = np.asarray(seq_lens, np.int32)
        ws = self._ws(self.lib.lobra_attn_workspace_bytes(lens, self.H))
        o = torch.empty_like(q)
        lse = torch.empty(self.H, q.shape[0], dtype=torch.float32, device=self.dev)
        self.lib.lobra_attn_fwd(lens, q, k, v, o, lse, ws)
        return o, lse, lens

    def backward(self, dO, q, k, v, o, lse, ctx, dq, dk, dv):
        lens = ctx
        ws = self._ws(self.lib.lobra_attn_bwd_workspace_bytes(lens, self.H, k.shape[-2]))
        self.lib.lobra_attn_bwd(lens, q, k, v, o, dO.contiguous(), lse, dq, dk, dv, ws)


def make_attention(backend: str, n_heads: int, head_dim: int, device, deterministic=False,
                   n_kv_heads: int | None = None):
    """q [T, n_heads, D]; k, v [T, n_kv_heads, D] (grouped-query attention when fewer)."""
    if backend == "cudnn":
        return CudnnVarlenAttention(n_heads, head_dim, device, n_kv_heads)
    if backend == "flash_attn":
        return FlashVarlenAttention(n_heads, head_dim, device, deterministic)
    if backend == "lobra":
        return LobraVarlenAttention(n_heads, head_dim, device, n_kv_heads)
    raise ValueError(f"unknown attention backend {backend!r}")
