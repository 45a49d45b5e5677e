"""One Llama-shaped decoder layer's seven LoRA projections driven through the C ABI.

This is plumbing around ``liblobra.so``: PyTorch allocates device memory, every step of
the hot path runs in the library's kernels.  Projections that read the same input (q/k/v,
gate/up) go through ``lobra_lora_group_fwd`` / ``lobra_lora_group_bwd`` (SURVEY §8(a) a1:
one pass over X for the shrinks and one for the dA reductions); o and down through
``lobra_lora_fwd`` / ``lobra_lora_bwd``.
Projections: q, k, v, gate, up are column-parallel and o, down
row-parallel under Megatron TP; every projection carries all tasks' adapters
(reading Q3).

Adapter gradients live in ONE flat fp32 buffer with the full-size layout on every rank
(DESIGN.md "Multi-GPU"): per projection dA_full [sum r, in_full] then dB_full
[out_full, sum r].  A TP rank writes only its partial sums into it (column rank: its dB
rows, partial dA; row rank: its dA column slice via dA_ld, partial dB), so one world
all-reduce (``lobra_adapter_allreduce``) yields the exact full gradients.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

# (name, in, out, tp kind, input group)
LLAMA2_7B = [("q", 4096, 4096, "col", "attn"), ("k", 4096, 4096, "col", "attn"),
             ("v", 4096, 4096, "col", "attn"), ("o", 4096, 4096, "row", "o_in"),
             ("gate", 4096, 11008, "col", "mlp"), ("up", 4096, 11008, "col", "mlp"),
             ("down", 11008, 4096, "row", "down_in")]
LLAMA2_70B = [("q", 8192, 8192, "col", "attn"), ("k", 8192, 1024, "col", "attn"),
              ("v", 8192, 1024, "col", "attn"), ("o", 8192, 8192, "row", "o_in"),
              ("gate", 8192, 28672, "col", "mlp"), ("up", 8192, 28672, "col", "mlp"),
              ("down", 28672, 8192, "row", "down_in")]


def algorithmic_flops(shapes, T: int, ranks, tokens_per_task=None) -> dict:
    """Algorithmic FLOPs of one fwd+bwd over T tokens: base
    4*T*sum(in*out) (no dW: frozen base), LoRA 6*sum_t T_t r_t sum(in+out)."""
    base = 4 * T * sum(i * o for _, i, o, *_ in shapes)
    if tokens_per_task is None:
        rt = T * float(np.mean(ranks))
    else:
        rt = float(sum(n * r for n, r in zip(tokens_per_task, ranks)))
    lora = 6 * rt * sum(i + o for _, i, o, *_ in shapes)
    return {"base": base, "lora": lora, "total": base + lora}


def shard(kind: str, tp_size: int, tp_rank: int, d_in: int, d_out: int):
    """Megatron TP slices of one projection: column-parallel shards `out`
    (W rows, B_t rows), row-parallel shards `in` (W columns, A_t columns)."""
    if kind == "col":
        o = d_out // tp_size
        return slice(0, d_in), slice(tp_rank * o, (tp_rank + 1) * o)
    i = d_in // tp_size
    return slice(tp_rank * i, (tp_rank + 1) * i), slice(0, d_out)


def grad_offsets(kind: str, tp_rank: int, in_l: int, out_l: int, d_in: int, rsum: int):
    """Where this rank writes its partial adapter gradients inside one projection's
    full-size [dA_full (rsum x d_in) | dB_full (d_out x rsum)] block of the flat buffer:
    (dA element offset, dA row stride, dB element offset).  Column rank: partial dA over
    its out-shard (full rows), its own dB rows.  Row rank: its dA column slice (row stride
    d_in), partial dB over its in-shard."""
    if kind == "row":
        return tp_rank * in_l, d_in, 0
    return 0, d_in, tp_rank * out_l * rsum


@dataclass
class _Proj:
    name: str
    d_in: int           # full widths
    d_out: int
    kind: str           # "col" | "row"
    group: str
    in_l: int           # local widths
    out_l: int
    W: torch.Tensor
    A: torch.Tensor
    B: torch.Tensor
    dA_off: int         # element offsets into the flat gradient buffer
    dB_off: int
    Hs: torch.Tensor | None = None


class LoraLayer:
    def __init__(self, shapes, ranks, scales, device, dtype=torch.bfloat16, tp_size=1, tp_rank=0,
                 comm=None, seed=0, group_inputs=True):
        self.device = torch.device(device)
        self.dtype = dtype
        self.code = _lib.dtype_code(dtype)
        self.ranks = np.asarray(ranks, np.int32)
        self.scales = np.asarray(scales, np.float32)
        self.rsum = int(self.ranks.sum())
        self.tp_size, self.tp_rank, self.comm = tp_size, tp_rank, comm
        self.group_inputs = group_inputs
        self.group_Hs = {}
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        self.projs = []
        off = 0
        for name, d_in, d_out, kind, group in shapes:
            if kind == "col":
                in_l, out_l = d_in, d_out // tp_size
            else:
                in_l, out_l = d_in // tp_size, d_out
            assert in_l * (tp_size if kind == "row" else 1) == d_in
            assert out_l * (tp_size if kind == "col" else 1) == d_out
            # full-size random init (synthetic weights), then the rank's shard
            W = self._randn((d_out, d_in), 1 / math.sqrt(d_in), g)
            A = self._randn((self.rsum, d_in), 1 / math.sqrt(d_in), g)
            Bparts = [self._randn((d_out, int(r)), 1 / math.sqrt(int(r)), g) for r in self.ranks]
            B = torch.cat(Bparts, dim=1)
            si, so = shard(kind, tp_size, tp_rank, d_in, d_out)
            W = W[so, si].contiguous()
            A = A[:, si].contiguous()
            B = B[so].contiguous()
            dA_off = off
            off += self.rsum * d_in
            dB_off = off
            off += d_out * self.rsum
            self.projs.append(_Proj(name, d_in, d_out, kind, group, in_l, out_l, W, A, B, dA_off, dB_off))
        self.flat_grad = torch.zeros(off, dtype=torch.float32, device=self.device)
        self.ws = torch.empty(0, dtype=torch.uint8, device=self.device)

    def relayout(self, ranks, scales):
        """New task set (ranks, scales) on the SAME frozen base: recompute the flat
        adapter-gradient layout and its offsets; the caller assigns the new A / B tensors
        ([sum r, in] / [out, sum r] local shards).  Used by the trainer when tasks join or
        leave."""
        self.ranks = np.asarray(ranks, np.int32)
        self.scales = np.asarray(scales, np.float32)
        self.rsum = int(self.ranks.sum())
        off = 0
        for p in self.projs:
            p.dA_off = off
            off += self.rsum * p.d_in
            p.dB_off = off
            off += p.d_out * self.rsum
            p.Hs = None
        self.group_Hs = {}
        self.flat_grad = torch.zeros(off, dtype=torch.float32, device=self.device)

    def _randn(self, shape, std, g):
        return (torch.randn(shape, generator=g, device=self.device, dtype=torch.float32) * std).to(self.dtype)

    # ------------------------------------------------------------------ buffers
    def input_width(self, group: str) -> int:
        for p in self.projs:
            if p.group == group:
                return p.in_l
        raise KeyError(group)

    def groups(self):
        seen = []
        for p in self.projs:
            if p.group not in seen:
                seen.append(p.group)
        return seen

    def alloc_io(self, T: int, seed: int = 1):
        """Synthetic activations X per input group and upstream grads dY per projection
        (values ~ N(0,1)); outputs Y / dX buffers."""
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        io = {"X": {}, "dY": {}, "Y": {}, "dX": {}}
        for grp in self.groups():
            w = self.input_width(grp)
            io["X"][grp] = torch.randn((T, w), generator=g, device=self.device).to(self.dtype)
            io["dX"][grp] = torch.empty((T, w), device=self.device, dtype=self.dtype)
        for p in self.projs:
            io["dY"][p.name] = torch.randn((T, p.out_l), generator=g, device=self.device).to(self.dtype)
            io["Y"][p.name] = torch.empty((T, p.out_l), device=self.device, dtype=self.dtype)
        return io

    def members(self, group: str):
        return [p for p in self.projs if p.group == group]

    def _grouped(self, group: str) -> bool:
        return self.group_inputs and len(self.members(group)) > 1

    def ensure(self, seq_lens, seq_task):
        self._ensure(seq_lens, seq_task)

    def _ensure(self, seq_lens, seq_task):
        need = 0
        for grp in self.groups():
            ms = self.members(grp)
            if self._grouped(grp):
                args = (self.code, ms[0].in_l, [p.out_l for p in ms], seq_lens, seq_task, self.ranks,
                        self.scales)
                need = max(need, _lib.lobra_lora_group_workspace_bytes(*args))
                hs = _lib.lobra_lora_group_saved_bytes(*args)
                if grp not in self.group_Hs or self.group_Hs[grp].numel() < hs:
                    self.group_Hs[grp] = torch.empty(hs, dtype=torch.uint8, device=self.device)
                continue
            for p in ms:
                need = max(need, _lib.lobra_lora_workspace_bytes(self.code, p.in_l, p.out_l, seq_lens,
                                                                 seq_task, self.ranks, self.scales))
                hs = _lib.lobra_lora_saved_bytes(self.code, p.in_l, p.out_l, seq_lens, seq_task,
                                                 self.ranks, self.scales)
                if p.Hs is None or p.Hs.numel() < hs:
                    p.Hs = torch.empty(hs, dtype=torch.uint8, device=self.device)
        if self.ws.numel() < need:
            self.ws = torch.empty(need, dtype=torch.uint8, device=self.device)

    def _grads(self, p):
        a_off, a_ld, b_off = grad_offsets(p.kind, self.tp_rank, p.in_l, p.out_l, p.d_in, self.rsum)
        fg = self.flat_grad
        dA = fg[p.dA_off + a_off:p.dA_off + self.rsum * p.d_in]
        dB = fg[p.dB_off + b_off:p.dB_off + p.d_out * self.rsum]
        return dA, dB, a_ld

    def _tp(self, p):
        if self.tp_size == 1 or self.comm is None:
            return _lib.LOBRA_TP_NONE, None
        return (_lib.LOBRA_TP_COLUMN if p.kind == "col" else _lib.LOBRA_TP_ROW), self.comm

    # ------------------------------------------------------------------ the hot path
    def forward_group(self, grp, seq_lens, seq_task, X, Ys: dict, stream=None):
        """The projections of input group `grp` over X [T, in] into Ys[name] [T, out]."""
        ms = self.members(grp)
        if self._grouped(grp):
            kind, comm = self._tp(ms[0])
            _lib.lobra_lora_group_fwd(X, [p.W for p in ms], [p.A for p in ms], [p.B for p in ms],
                                      self.ranks, self.scales, seq_lens, seq_task, [Ys[p.name] for p in ms],
                                      self.group_Hs[grp], self.ws, tp_kind=kind, comm=comm, stream=stream)
            return
        for p in ms:
            kind, comm = self._tp(p)
            _lib.lobra_lora_fwd(X, p.W, p.A, p.B, self.ranks, self.scales, seq_lens, seq_task, Ys[p.name], p.Hs,
                                self.ws, tp_kind=kind, comm=comm, stream=stream)

    def backward_group(self, grp, seq_lens, seq_task, X, dYs: dict, dX, accumulate_dadb: bool, stream=None):
        """A group's projections sum into one dX (the group call, or accumulate_dx on the
        single calls); for column-parallel TP the dX all-reduce runs once per group, after
        its last projection, and then sums every projection's partial."""
        ms = self.members(grp)
        if self._grouped(grp):
            kind, comm = self._tp(ms[0])
            gr = [self._grads(p) for p in ms]
            _lib.lobra_lora_group_bwd(X, [p.W for p in ms], [p.A for p in ms], [p.B for p in ms], self.ranks,
                                      self.scales, seq_lens, seq_task, self.group_Hs[grp],
                                      [dYs[p.name] for p in ms], dX, [g[0] for g in gr], [g[1] for g in gr],
                                      self.ws, accumulate_dadb=accumulate_dadb, dA_ld=gr[0][2], tp_kind=kind,
                                      comm=comm, stream=stream)
            return
        for i, p in enumerate(ms):
            kind, comm = self._tp(p)
            if kind == _lib.LOBRA_TP_COLUMN and i != len(ms) - 1:
                kind, comm = _lib.LOBRA_TP_NONE, None
            dA, dB, dA_ld = self._grads(p)
            _lib.lobra_lora_bwd(X, p.W, p.A, p.B, self.ranks, self.scales, seq_lens, seq_task, p.Hs, dYs[p.name],
                                dX, dA, dB, self.ws, accumulate_dx=i > 0, accumulate_dadb=accumulate_dadb,
                                dA_ld=dA_ld, tp_kind=kind, comm=comm, stream=stream)

    def forward(self, seq_lens, seq_task, io, T: int, stream=None):
        """Every projection on synthetic per-group inputs io["X"][group] (the north-star
        step: the seven projections of one layer)."""
        self._ensure(seq_lens, seq_task)
        for grp in self.groups():
            self.forward_group(grp, seq_lens, seq_task, io["X"][grp][:T],
                               {p.name: io["Y"][p.name][:T] for p in self.members(grp)}, stream)

    def backward(self, seq_lens, seq_task, io, T: int, accumulate_dadb: bool, stream=None):
        for grp in self.groups():
            self.backward_group(grp, seq_lens, seq_task, io["X"][grp][:T],
                                {p.name: io["dY"][p.name][:T] for p in self.members(grp)}, io["dX"][grp][:T],
                                accumulate_dadb, stream)

    def sync_adapter_grads(self, stream=None):
        if self.comm is not None and self.comm.world > 1:
            _lib.lobra_adapter_allreduce(self.comm, self.flat_grad, stream=stream)
