"""Pins of the fp64 LoRA oracle against what the paper and mathematics fix
(not against itself).  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import lora as O
from workloads import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _tiny(seed=0, T_lens=(5, 3, 7, 4), tasks=(0, 1, 0, 2), ranks=(3, 2, 4), d_in=6, d_out=5):
    rng = np.random.default_rng(seed)
    lens = np.array(T_lens, np.int32)
    tids = np.array(tasks, np.int32)
    T = int(lens.sum())
    R = int(sum(ranks))
    X = rng.standard_normal((T, d_in))
    W = rng.standard_normal((d_out, d_in))
    A = rng.standard_normal((R, d_in))
    B = rng.standard_normal((d_out, R))
    dY = rng.standard_normal((T, d_out))
    s = np.array([1.7, -0.5, 2.0])[:len(ranks)]
    return X, W, A, B, list(ranks), s, lens, tids, dY


def test_golden_hand_example():
    """Hand-worked integer example (tests/golden/lora_tiny.json)."""
    g = json.load(open(os.path.join(GOLD, "lora_tiny.json")))
    args = (np.array(g["x"], float), np.array(g["W"], float), np.array(g["A"], float),
            np.array(g["B"], float), [g["rank"]], [g["scale"]], [1], [0])
    Y = O.lora_fwd(*args)
    assert np.array_equal(Y, np.array(g["y"], float))
    dX, dA, dB = O.lora_bwd(*args, np.array(g["dy"], float))
    assert np.array_equal(dX, np.array(g["dx"], float))
    assert np.array_equal(dA, np.array(g["dA"], float))
    assert np.array_equal(dB, np.array(g["dB"], float))


def test_B_zero_gives_base_exactly():
    """North-star pin: B_t = 0 => Y = X W^T bit for bit."""
    X, W, A, B, r, s, lens, tids, _ = _tiny(1)
    Y = O.lora_fwd(X, W, A, np.zeros_like(B), r, s, lens, tids)
    assert np.array_equal(Y, X @ W.T)


def test_merged_weight():
    """North-star pin: running with the merged weight W + s_t B_t A_t gives the same Y."""
    X, W, A, B, r, s, lens, tids, _ = _tiny(2)
    Y = O.lora_fwd(X, W, A, B, r, s, lens, tids)
    roff = np.concatenate([[0], np.cumsum(r)])
    off = 0
    for L, t in zip(lens, tids):
        Wm = W + s[t] * B[:, roff[t]:roff[t + 1]] @ A[roff[t]:roff[t + 1]]
        ref = X[off:off + L] @ Wm.T
        assert np.max(np.abs(Y[off:off + L] - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
        off += L


def _loss(X, W, A, B, r, s, lens, tids, Rm):
    Y = O.lora_fwd(X, W, A, B, r, s, lens, tids)
    return 0.5 * np.sum(Y * Y) + np.sum(Y * Rm)


@pytest.mark.parametrize("seed", [3, 4])
def test_finite_differences(seed):
    """North-star pin: central differences on L = 1/2|Y|^2 + <Y,R> (dY = Y + R).
    L is quadratic in each of X, A_t, B_t separately, so central differences are exact
    up to rounding."""
    X, W, A, B, r, s, lens, tids, Rm = _tiny(seed)
    Y = O.lora_fwd(X, W, A, B, r, s, lens, tids)
    dX, dA, dB = O.lora_bwd(X, W, A, B, r, s, lens, tids, Y + Rm)
    h = 1e-3
    for name, P, G in (("X", X, dX), ("A", A, dA), ("B", B, dB)):
        num = np.zeros_like(P)
        for idx in np.ndindex(P.shape):
            Pp, Pm = P.copy(), P.copy()
            Pp[idx] += h
            Pm[idx] -= h
            kw = {"X": X, "A": A, "B": B}
            kp, km = dict(kw), dict(kw)
            kp[name], km[name] = Pp, Pm
            num[idx] = (_loss(kp["X"], W, kp["A"], kp["B"], r, s, lens, tids, Rm)
                        - _loss(km["X"], W, km["A"], km["B"], r, s, lens, tids, Rm)) / (2 * h)
        err = np.max(np.abs(num - G)) / np.max(np.abs(G))
        assert err < 1e-9, (name, err)


def test_torch_autograd():
    """Independent library cross-check: torch fp64 autograd of the dense per-sequence
    formula y = x W^T + s (x A^T) B^T."""
    torch = pytest.importorskip("torch")
    X, W, A, B, r, s, lens, tids, dY = _tiny(5)
    roff = np.concatenate([[0], np.cumsum(r)])
    tX = torch.tensor(X, requires_grad=True)
    tA = torch.tensor(A, requires_grad=True)
    tB = torch.tensor(B, requires_grad=True)
    tW = torch.tensor(W)
    outs, off = [], 0
    for L, t in zip(lens, tids):
        x = tX[off:off + L]
        a = tA[roff[t]:roff[t + 1]]
        b = tB[:, roff[t]:roff[t + 1]]
        outs.append(torch.nn.functional.linear(x, tW) + s[t] * torch.nn.functional.linear(
            torch.nn.functional.linear(x, a), b))
        off += L
    Yt = torch.cat(outs)
    Yt.backward(torch.tensor(dY))
    Y = O.lora_fwd(X, W, A, B, r, s, lens, tids)
    dX, dA, dB = O.lora_bwd(X, W, A, B, r, s, lens, tids, dY)
    assert np.max(np.abs(Y - Yt.detach().numpy())) < 1e-12
    assert np.max(np.abs(dX - tX.grad.numpy())) < 1e-12
    assert np.max(np.abs(dA - tA.grad.numpy())) < 1e-12
    assert np.max(np.abs(dB - tB.grad.numpy())) < 1e-12


def test_loops_equal_numpy_on_c1():
    """Tiny brute force: the pure-loop implementation equals the NumPy one on C1."""
    wl = synth.config_c1()
    t = synth.layer_tensors(wl, 64, 64, seed=1)
    # use a subset of sequences to keep the pure-Python loops to a few seconds
    lens, tids = wl.seq_lens[:3], wl.seq_task[:3]
    T = int(lens.sum())
    args = (t["X"][:T], t["W"], t["A"], t["B"], wl.ranks.tolist(), wl.scales, lens, tids)
    Y = O.lora_fwd(*args)
    Yl = O.lora_fwd_loops(*args)
    assert np.max(np.abs(Y - Yl)) <= 1e-13 * np.max(np.abs(Y))
    g = O.lora_bwd(*args, t["dY"][:T])
    gl = O.lora_bwd_loops(*args, t["dY"][:T])
    for a, b in zip(g, gl):
        assert np.max(np.abs(a - b)) <= 1e-13 * np.max(np.abs(a))


def test_packing_order_invariance():
    """A permutation of the sequences leaves per-sequence Y and dX bitwise equal and
    dA/dB equal to 1e-12 (packed rows are independent)."""
    X, W, A, B, r, s, lens, tids, dY = _tiny(6, T_lens=(5, 3, 7, 4, 2, 6), tasks=(0, 1, 0, 2, 1, 2))
    offs = np.concatenate([[0], np.cumsum(lens)])
    perm = np.array([3, 0, 5, 2, 1, 4])
    rows = np.concatenate([np.arange(offs[k], offs[k + 1]) for k in perm])
    Y = O.lora_fwd(X, W, A, B, r, s, lens, tids)
    Yp = O.lora_fwd(X[rows], W, A, B, r, s, lens[perm], tids[perm])
    assert np.array_equal(Y[rows], Yp)
    dX, dA, dB = O.lora_bwd(X, W, A, B, r, s, lens, tids, dY)
    dXp, dAp, dBp = O.lora_bwd(X[rows], W, A, B, r, s, lens[perm], tids[perm], dY[rows])
    assert np.array_equal(dX[rows], dXp)
    assert np.max(np.abs(dA - dAp)) <= 1e-12 * np.max(np.abs(dA))
    assert np.max(np.abs(dB - dBp)) <= 1e-12 * np.max(np.abs(dB))


def test_special_cases():
    X, W, A, B, r, s, lens, tids, dY = _tiny(7)
    # s_t = 0 => base
    Y0 = O.lora_fwd(X, W, A, B, r, np.zeros(3), lens, tids)
    assert np.array_equal(Y0, X @ W.T)
    # W = 0 => pure adapter path (dense textbook chain)
    Yw = O.lora_fwd(X, np.zeros_like(W), A, B, r, s, lens, tids)
    roff = np.concatenate([[0], np.cumsum(r)])
    off = 0
    for L, t in zip(lens, tids):
        ref = s[t] * (X[off:off + L] @ A[roff[t]:roff[t + 1]].T) @ B[:, roff[t]:roff[t + 1]].T
        assert np.max(np.abs(Yw[off:off + L] - ref)) <= 1e-13 * max(1, np.max(np.abs(ref)))
        off += L
    # a task with no tokens => zero gradient blocks (task 2 absent)
    t3 = np.array([0, 1, 0, 1], np.int32)
    _, dA, dB = O.lora_bwd(X, W, A, B, r, s, lens, t3, dY)
    assert not dA[roff[2]:roff[3]].any() and not dB[:, roff[2]:roff[3]].any()
    # linearity in dY
    g1 = O.lora_bwd(X, W, A, B, r, s, lens, tids, dY)
    g2 = O.lora_bwd(X, W, A, B, r, s, lens, tids, 3.0 * dY)
    for a, b in zip(g1, g2):
        assert np.max(np.abs(3.0 * a - b)) <= 1e-12 * np.max(np.abs(b))
    # accumulating over two halves of the batch equals the whole (gradient accumulation,
    # P:257-259)
    h = 2
    offs = np.concatenate([[0], np.cumsum(lens)])
    a1 = O.lora_bwd(X[:offs[h]], W, A, B, r, s, lens[:h], tids[:h], dY[:offs[h]])
    a2 = O.lora_bwd(X[offs[h]:], W, A, B, r, s, lens[h:], tids[h:], dY[offs[h]:])
    assert np.max(np.abs(a1[1] + a2[1] - g1[1])) <= 1e-12 * np.max(np.abs(g1[1]))
    assert np.max(np.abs(a1[2] + a2[2] - g1[2])) <= 1e-12 * np.max(np.abs(g1[2]))
    # single task, single sequence = dense LoRA
    X1 = X[:5]
    Y1 = O.lora_fwd(X1, W, A, B, r, s, [5], [1])
    ref = X1 @ W.T + s[1] * (X1 @ A[3:5].T) @ B[:, 3:5].T
    assert np.max(np.abs(Y1 - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_max_rel_err_definition():
    assert O.max_rel_err([1.0, 2.0], [1.0, 2.0]) == 0.0
    assert O.max_rel_err([1.0, 2.5], [1.0, 2.0]) == 0.25
    assert O.max_rel_err([0.0], [0.0]) == 0.0
