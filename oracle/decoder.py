"""fp64 oracle of one Llama decoder layer with multi-task LoRA on its seven projections
-- TEST INFRASTRUCTURE ONLY.

Scope: the full fine-tuning step of one layer that the paper's cost model profiles
(App. D: "the running time of the attention mechanism is proportional to the
square of s, whilst for other modules, it is proportional to s ... we simplify and
expedite the offline process by profiling only a single layer").  The paper fine-tunes
Llama2-7B / Qwen2.5-32B / Llama2-70B and gives no layer formulas; the layer below
is the public Llama-2 definition (reading Q27): pre-norm RMSNorm (eps 1e-5),
rotary embeddings (theta 10000, rotate-half pairing (j, j + D/2)) restarted at position 0
in every packed sequence, causal attention restricted to each sequence (block-diagonal
mask over the packed batch, "pack ... without cross-contamination"), SwiGLU MLP,
two residual adds.  The frozen base (W, norm gains) gets no gradient; the
LoRA adapters of all seven projections do (oracle.lora, reading Q3).

Each function is the plain definition written out with NumPy (matmul / exp are the only
library primitives); the backward is the chain rule written out step by step.
"""
from __future__ import annotations

import numpy as np

from . import lora as L

PROJS = ("q", "k", "v", "o", "gate", "up", "down")


# ------------------------------------------------------------------ building blocks
def rmsnorm(x, g, eps):
    """y = x / sqrt(mean(x^2) + eps) * g, per row; returns (y, rstd)."""
    x = np.asarray(x, np.float64)
    rstd = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return x * rstd * np.asarray(g, np.float64), rstd[..., 0]


def rmsnorm_bwd(dy, x, g, eps):
    """d/dx of rmsnorm with frozen g:  with u = g * dy and r = rstd,
    dx = r u - x r^3 (u . x) / n."""
    x = np.asarray(x, np.float64)
    u = np.asarray(dy, np.float64) * np.asarray(g, np.float64)
    n = x.shape[-1]
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return r * u - x * r ** 3 * np.sum(u * x, axis=-1, keepdims=True) / n


def positions(seq_lens):
    """Token position inside its own sequence (restarts at 0 per packed sequence)."""
    return np.concatenate([np.arange(int(n)) for n in seq_lens] or [np.zeros(0, int)]).astype(np.int64)


def rope(x, pos, theta, inverse=False):
    """Rotary embedding on x [T, H, D] (rotate-half pairing (j, j + D/2)):
    angle_j = pos * theta^(-2j/D);  (a, b) -> (a cos - b sin, b cos + a sin).
    inverse=True rotates by -angle (the transpose: the backward of rope)."""
    x = np.asarray(x, np.float64)
    D = x.shape[-1]
    j = np.arange(D // 2, dtype=np.float64)
    ang = np.asarray(pos, np.float64)[:, None] * theta ** (-2.0 * j / D)      # [T, D/2]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    if inverse:
        s = -s
    a, b = x[..., : D // 2], x[..., D // 2:]
    return np.concatenate([a * c - b * s, b * c + a * s], axis=-1)


def _kv_heads(x, H):
    """Grouped-query attention (Llama-2-70B): query head i reads kv head i // (H / H_kv)."""
    return np.repeat(x, H // x.shape[1], axis=1)


def attention(q, k, v, seq_lens):
    """Causal softmax attention inside every packed sequence; q [T, H, D], k, v [T, H_kv, D]
    with H_kv | H (H_kv = H: multi-head).  Returns (O [T, H, D], P list per sequence
    [H, n, n])."""
    q, k, v = (np.asarray(a, np.float64) for a in (q, k, v))
    k, v = _kv_heads(k, q.shape[1]), _kv_heads(v, q.shape[1])
    D = q.shape[-1]
    O = np.zeros_like(q)
    Ps = []
    off = 0
    for n in (int(x) for x in seq_lens):
        sl = slice(off, off + n)
        qs, ks, vs = q[sl].transpose(1, 0, 2), k[sl].transpose(1, 0, 2), v[sl].transpose(1, 0, 2)
        S = qs @ ks.transpose(0, 2, 1) / np.sqrt(D)                     # [H, n, n]
        S = np.where(np.tril(np.ones((n, n), bool))[None], S, -np.inf)
        S = S - S.max(axis=-1, keepdims=True)
        P = np.exp(S)
        P = P / P.sum(axis=-1, keepdims=True)
        O[sl] = (P @ vs).transpose(1, 0, 2)
        Ps.append(P)
        off += n
    return O, Ps


def attention_bwd(dO, q, k, v, Ps, seq_lens):
    """dV = P^T dO; dP = dO V^T; dS = P * (dP - rowsum(dP * P)); dQ = dS K / sqrt(D);
    dK = dS^T Q / sqrt(D)  (per sequence and query head; with grouped kv heads the dK, dV
    of a kv head sum over the query heads that read it)."""
    dO, q, k, v = (np.asarray(a, np.float64) for a in (dO, q, k, v))
    Hkv = k.shape[1]
    k, v = _kv_heads(k, q.shape[1]), _kv_heads(v, q.shape[1])
    D = q.shape[-1]
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    off = 0
    for n, P in zip((int(x) for x in seq_lens), Ps):
        sl = slice(off, off + n)
        qs, ks, vs = q[sl].transpose(1, 0, 2), k[sl].transpose(1, 0, 2), v[sl].transpose(1, 0, 2)
        g = dO[sl].transpose(1, 0, 2)
        dV = P.transpose(0, 2, 1) @ g
        dP = g @ vs.transpose(0, 2, 1)
        dS = P * (dP - np.sum(dP * P, axis=-1, keepdims=True))
        dq[sl] = (dS @ ks / np.sqrt(D)).transpose(1, 0, 2)
        dk[sl] = (dS.transpose(0, 2, 1) @ qs / np.sqrt(D)).transpose(1, 0, 2)
        dv[sl] = dV.transpose(1, 0, 2)
        off += n
    T, H = dk.shape[0], dk.shape[1]
    g = H // Hkv
    return dq, dk.reshape(T, Hkv, g, D).sum(axis=2), dv.reshape(T, Hkv, g, D).sum(axis=2)


def silu(x):
    return x / (1.0 + np.exp(-x))


def swiglu(gate, up):
    gate, up = np.asarray(gate, np.float64), np.asarray(up, np.float64)
    return silu(gate) * up


def swiglu_bwd(d, gate, up):
    """act = silu(g) u:  d_up = d silu(g);  d_gate = d u sigma(g) (1 + g (1 - sigma(g)))."""
    d, gate, up = (np.asarray(a, np.float64) for a in (d, gate, up))
    sg = 1.0 / (1.0 + np.exp(-gate))
    return d * up * sg * (1.0 + gate * (1.0 - sg)), d * gate * sg


# ------------------------------------------------------------------ the layer
def layer_fwd(X, P, cfg, ranks, scales, seq_lens, seq_task):
    """One Llama decoder layer over the packed batch X [T, h].  P: dict with g_attn,
    g_mlp and, per projection p, (W_p, A_p, B_p).  cfg: n_heads, eps, theta (n_kv_heads:
    from the k projection's width).  Returns (Y, cache)."""
    H, eps, theta = cfg["n_heads"], cfg["eps"], cfg["theta"]
    X = np.asarray(X, np.float64)
    T, h = X.shape
    D = h // H
    lo = lambda Z, p: L.lora_fwd(Z, P[p][0], P[p][1], P[p][2], ranks, scales, seq_lens, seq_task)
    h1, _ = rmsnorm(X, P["g_attn"], eps)
    q, k, v = lo(h1, "q"), lo(h1, "k"), lo(h1, "v")
    Hkv = k.shape[1] // D
    pos = positions(seq_lens)
    qr = rope(q.reshape(T, H, D), pos, theta)
    kr = rope(k.reshape(T, Hkv, D), pos, theta)
    vv = v.reshape(T, Hkv, D)
    att, Ps = attention(qr, kr, vv, seq_lens)
    att = att.reshape(T, h)
    o = lo(att, "o")
    x2 = X + o
    h2, _ = rmsnorm(x2, P["g_mlp"], eps)
    gate, up = lo(h2, "gate"), lo(h2, "up")
    act = swiglu(gate, up)
    down = lo(act, "down")
    Y = x2 + down
    cache = dict(X=X, h1=h1, q=q, k=k, v=v, qr=qr, kr=kr, vv=vv, Ps=Ps, att=att, x2=x2, h2=h2,
                 gate=gate, up=up, act=act, pos=pos)
    return Y, cache


def layer_bwd(dY, P, cfg, ranks, scales, seq_lens, seq_task, cache):
    """Backward of layer_fwd given dY: returns (dX, grads) with grads[p] = (dA_p, dB_p)."""
    H, eps, theta = cfg["n_heads"], cfg["eps"], cfg["theta"]
    c = cache
    T, h = c["X"].shape
    D = h // H
    dY = np.asarray(dY, np.float64)
    grads = {}

    def lb(Z, p, d):
        dZ, dA, dB = L.lora_bwd(Z, P[p][0], P[p][1], P[p][2], ranks, scales, seq_lens, seq_task, d)
        grads[p] = (dA, dB)
        return dZ

    d_act = lb(c["act"], "down", dY)                          # y = x2 + down
    d_gate, d_up = swiglu_bwd(d_act, c["gate"], c["up"])
    dh2 = lb(c["h2"], "gate", d_gate) + lb(c["h2"], "up", d_up)
    dx2 = dY + rmsnorm_bwd(dh2, c["x2"], P["g_mlp"], eps)     # x2 feeds y and h2
    d_att = lb(c["att"], "o", dx2)
    dqr, dkr, dv = attention_bwd(d_att.reshape(T, H, D), c["qr"], c["kr"], c["vv"], c["Ps"], seq_lens)
    dq = rope(dqr, c["pos"], theta, inverse=True).reshape(T, h)
    dk = rope(dkr, c["pos"], theta, inverse=True).reshape(T, -1)
    dh1 = lb(c["h1"], "q", dq) + lb(c["h1"], "k", dk) + lb(c["h1"], "v", dv.reshape(T, -1))
    dX = dx2 + rmsnorm_bwd(dh1, c["X"], P["g_attn"], eps)      # X feeds x2 and h1
    return dX, grads
