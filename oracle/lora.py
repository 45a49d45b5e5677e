"""fp64 oracle of the multi-task LoRA layer -- TEST INFRASTRUCTURE ONLY.

What it computes (the plain definition; DESIGN.md §Readings Q1, Q2, Q7, Q24):

  PAPER.md P:231 (§2.1): "For a model weight matrix W in R^{in x out}, LoRA trains two
  low-rank matrices A in R^{r x out}, B in R^{in x r} ... and computes XW + XBA."
  P:135: the inputs of all tasks are fused into one batch; the base op is batched, the
  per-task adapters run as "customized operations".  P:261-266: sequences are packed.

With the north-star names (paper's B = our A_t "shrink", paper's A = our B_t "expand")
and PyTorch/PEFT storage (W [out,in], A_t [r_t,in], B_t [out,r_t]), every token row x
of a sequence whose task is t computes

    y = x W^T + s_t (x A_t^T) B_t^T

and, given the upstream gradient dy (W is frozen, P:74, P:230 -> no dW):

    dx   = dy W + s_t (dy B_t) A_t
    dA_t = s_t * sum_{rows of t} (dy B_t)^T x        ([r_t, in])
    dB_t = s_t * sum_{rows of t} dy^T (x A_t^T)       ([out, r_t])

Gradient sums are plain sums over tokens (reading Q7).  Inputs are the exact values
the GPU receives, widened to fp64.  Rows are independent, so the per-sequence loop
below *is* the definition; np.matmul is the only library primitive used.

Adapter storage follows the C ABI: A_cat [sum_t r_t, in] with task t's rows at
roff[t] = sum_{u<t} r_u, and B_cat [out, sum_t r_t] with task t's columns at roff[t].
"""
from __future__ import annotations

import numpy as np


def _roff(ranks) -> np.ndarray:
    ranks = np.asarray(ranks, dtype=np.int64)
    return np.concatenate([[0], np.cumsum(ranks)]).astype(np.int64)


def _segments(seq_lens, seq_task):
    """Yield (row_start, row_end, task) per sequence, in packing order."""
    off = 0
    for L, t in zip(np.asarray(seq_lens).tolist(), np.asarray(seq_task).tolist()):
        yield off, off + int(L), int(t)
        off += int(L)


def lora_fwd(X, W, A_cat, B_cat, ranks, scales, seq_lens, seq_task, return_h=False):
    """Y [T,out] = per sequence: X_k W^T + s_t (X_k A_t^T) B_t^T.

    If ``return_h``, also returns H [T, max r] with H_k = s_t X_k A_t^T (the pre-scaled
    shrink output, zero-padded on the right), for diagnostics."""
    X = np.asarray(X, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    A_cat = np.asarray(A_cat, dtype=np.float64)
    B_cat = np.asarray(B_cat, dtype=np.float64)
    roff = _roff(ranks)
    T = X.shape[0]
    Y = np.zeros((T, W.shape[0]), dtype=np.float64)
    rmax = int(max(ranks)) if len(ranks) else 0
    H = np.zeros((T, rmax), dtype=np.float64)
    for a, b, t in _segments(seq_lens, seq_task):
        if b == a:
            continue
        x = X[a:b]
        At = A_cat[roff[t]:roff[t + 1]]          # [r, in]
        Bt = B_cat[:, roff[t]:roff[t + 1]]       # [out, r]
        s = float(scales[t])
        base = np.matmul(x, W.T)
        xa = np.matmul(x, At.T)                  # [len, r]
        Y[a:b] = base + s * np.matmul(xa, Bt.T)
        H[a:b, :At.shape[0]] = s * xa
    return (Y, H) if return_h else Y


def lora_bwd(X, W, A_cat, B_cat, ranks, scales, seq_lens, seq_task, dY, want_dx=True):
    """Returns (dX [T,in], dA_cat [sum r, in], dB_cat [out, sum r]) -- see module doc.
    ``want_dx=False`` skips dX (returned as None) for large adapter-gradient checks."""
    X = np.asarray(X, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    A_cat = np.asarray(A_cat, dtype=np.float64)
    B_cat = np.asarray(B_cat, dtype=np.float64)
    dY = np.asarray(dY, dtype=np.float64)
    roff = _roff(ranks)
    dX = np.zeros_like(X) if want_dx else None
    dA = np.zeros_like(A_cat)
    dB = np.zeros_like(B_cat)
    for a, b, t in _segments(seq_lens, seq_task):
        if b == a:
            continue
        x, dy = X[a:b], dY[a:b]
        At = A_cat[roff[t]:roff[t + 1]]
        Bt = B_cat[:, roff[t]:roff[t + 1]]
        s = float(scales[t])
        g = np.matmul(dy, Bt)                    # dy B_t        [len, r]
        if want_dx:
            dX[a:b] = np.matmul(dy, W) + s * np.matmul(g, At)
        dA[roff[t]:roff[t + 1]] += s * np.matmul(g.T, x)
        dB[:, roff[t]:roff[t + 1]] += s * np.matmul(dy.T, np.matmul(x, At.T))
    return dX, dA, dB


# ---------------------------------------------------------------------------
# Pure-Python loop version for tiny inputs (cross-checks the NumPy version).
# ---------------------------------------------------------------------------
def lora_fwd_loops(X, W, A_cat, B_cat, ranks, scales, seq_lens, seq_task):
    X = [[float(v) for v in row] for row in np.asarray(X)]
    W = np.asarray(W, dtype=np.float64).tolist()
    A = np.asarray(A_cat, dtype=np.float64).tolist()
    B = np.asarray(B_cat, dtype=np.float64).tolist()
    roff = _roff(ranks).tolist()
    n_in, n_out = len(W[0]), len(W)
    Y = [[0.0] * n_out for _ in X]
    for a, b, t in _segments(seq_lens, seq_task):
        s = float(scales[t])
        for i in range(a, b):
            xa = [sum(X[i][k] * A[roff[t] + q][k] for k in range(n_in)) for q in range(ranks[t])]
            for o in range(n_out):
                base = sum(X[i][k] * W[o][k] for k in range(n_in))
                lora = sum(xa[q] * B[o][roff[t] + q] for q in range(ranks[t]))
                Y[i][o] = base + s * lora
    return np.array(Y)


def lora_bwd_loops(X, W, A_cat, B_cat, ranks, scales, seq_lens, seq_task, dY):
    X = np.asarray(X, dtype=np.float64).tolist()
    W = np.asarray(W, dtype=np.float64).tolist()
    A = np.asarray(A_cat, dtype=np.float64).tolist()
    B = np.asarray(B_cat, dtype=np.float64).tolist()
    dY = np.asarray(dY, dtype=np.float64).tolist()
    roff = _roff(ranks).tolist()
    n_in, n_out = len(W[0]), len(W)
    R = roff[-1]
    dX = [[0.0] * n_in for _ in X]
    dA = [[0.0] * n_in for _ in range(R)]
    dB = [[0.0] * R for _ in range(n_out)]
    for a, b, t in _segments(seq_lens, seq_task):
        s = float(scales[t])
        r = int(ranks[t])
        for i in range(a, b):
            g = [sum(dY[i][o] * B[o][roff[t] + q] for o in range(n_out)) for q in range(r)]
            xa = [sum(X[i][k] * A[roff[t] + q][k] for k in range(n_in)) for q in range(r)]
            for k in range(n_in):
                dX[i][k] = (sum(dY[i][o] * W[o][k] for o in range(n_out))
                            + s * sum(g[q] * A[roff[t] + q][k] for q in range(r)))
            for q in range(r):
                for k in range(n_in):
                    dA[roff[t] + q][k] += s * g[q] * X[i][k]
                for o in range(n_out):
                    dB[o][roff[t] + q] += s * dY[i][o] * xa[q]
    return np.array(dX), np.array(dA), np.array(dB)


def max_rel_err(got, ref) -> float:
    """Reading Q9: err = max|g - o| / max|o| over one output tensor (0 if both are zero)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = float(np.max(np.abs(ref))) if ref.size else 0.0
    num = float(np.max(np.abs(got - ref))) if ref.size else 0.0
    if den == 0.0:
        return num
    return num / den
