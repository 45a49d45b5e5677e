"""GPU parity of the decoder-layer elementwise ops (RMSNorm, RoPE, SwiGLU)
through the C ABI against the fp64 oracle (oracle/decoder.py) on the same bf16 inputs.

Tolerance: one bf16 rounding of every output (relative 2^-9) on top of fp32 arithmetic;
metric max|gpu - oracle| / max|oracle| <= 1e-2 (reading Q9).  The fused residual sum
S = X + R is checked bitwise (fp32 add of two bf16 values is exact, then one RNE).
"""
import numpy as np
import pytest

from oracle import decoder as Dd
from oracle import lora as O
from workloads import synth

pytestmark = pytest.mark.gpu
TOL = 1e-2


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _bf(a):
    return synth.round_bf16(np.asarray(a)).astype(np.float64)


def _up(torch, a):
    return torch.from_numpy(np.ascontiguousarray(synth.round_bf16(np.asarray(a)))).cuda().to(torch.bfloat16)


def _np(x):
    return x.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("T,h,resid", [(37, 4096, False), (37, 4096, True), (5, 8192, True), (9, 64, False)])
def test_rmsnorm_fwd_bwd(T, h, resid):
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    rng = np.random.default_rng(h + T)
    X = rng.standard_normal((T, h)) * 2
    R = rng.standard_normal((T, h)) if resid else None
    g = 1 + 0.2 * rng.standard_normal(h)
    dY = rng.standard_normal((T, h))
    dRes = rng.standard_normal((T, h)) if resid else None
    Xd, gd, dYd = _up(torch, X), _up(torch, g), _up(torch, dY)
    Rd = _up(torch, R) if resid else None
    S = torch.empty_like(Xd) if resid else None
    Y = torch.empty_like(Xd)
    rstd = torch.empty(T, device="cuda", dtype=torch.float32)
    _lib.lobra_rmsnorm_fwd(Xd, gd, 1e-5, Y, rstd, R=Rd, S_out=S)
    Sref = _bf(_bf(X) + _bf(R)) if resid else _bf(X)
    if resid:
        assert np.array_equal(_np(S), Sref)
    Yo, ro = Dd.rmsnorm(Sref, _bf(g), 1e-5)
    assert O.max_rel_err(_np(Y), Yo) <= TOL
    assert np.allclose(rstd.cpu().numpy(), ro, rtol=1e-5)
    dS = torch.empty_like(Xd)
    _lib.lobra_rmsnorm_bwd(dYd, S if resid else Xd, gd, rstd, dS, dRes=_up(torch, dRes) if resid else None)
    ref = Dd.rmsnorm_bwd(_bf(dY), Sref, _bf(g), 1e-5) + (_bf(dRes) if resid else 0)
    assert O.max_rel_err(_np(dS), ref) <= TOL


@pytest.mark.parametrize("inverse", [False, True])
def test_rope_packed_positions(inverse):
    """Q and K as strided column blocks of one [T, 3 h] qkv buffer; positions restart per
    sequence (lengths 1, 700, 33, 2048: > 1K-position angles, a 1-token sequence)."""
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    lens = [1, 700, 33, 2048]
    T, H, D = sum(lens), 4, 128
    rng = np.random.default_rng(3)
    qkv = rng.standard_normal((T, 3 * H * D))
    buf = _up(torch, qkv)
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    q, k = buf[:, :H * D], buf[:, H * D:2 * H * D]
    _lib.lobra_rope(cu, T, H, D, 10000.0, q, k, inverse=inverse)
    pos = Dd.positions(lens)
    for part, sl in ((q, slice(0, H * D)), (k, slice(H * D, 2 * H * D))):
        ref = Dd.rope(_bf(qkv[:, sl]).reshape(T, H, D), pos, 10000.0, inverse=inverse).reshape(T, H * D)
        assert O.max_rel_err(_np(part), ref) <= TOL
    assert np.array_equal(_np(buf[:, 2 * H * D:]), _bf(qkv[:, 2 * H * D:]))   # v untouched
    # forward then inverse returns the input to bf16 rounding
    _lib.lobra_rope(cu, T, H, D, 10000.0, q, k, inverse=not inverse)
    assert O.max_rel_err(_np(buf[:, :H * D]), _bf(qkv[:, :H * D])) <= TOL


def test_swiglu_fwd_bwd():
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    rng = np.random.default_rng(4)
    n = (333, 11008)
    g, u, d = rng.standard_normal(n) * 3, rng.standard_normal(n), rng.standard_normal(n)
    gd, ud, dd = _up(torch, g), _up(torch, u), _up(torch, d)
    act = torch.empty_like(gd)
    _lib.lobra_swiglu_fwd(gd, ud, act)
    assert O.max_rel_err(_np(act), Dd.swiglu(_bf(g), _bf(u))) <= TOL
    dg, du = torch.empty_like(gd), torch.empty_like(gd)
    _lib.lobra_swiglu_bwd(dd, gd, ud, dg, du)
    rg, ru = Dd.swiglu_bwd(_bf(d), _bf(g), _bf(u))
    assert O.max_rel_err(_np(dg), rg) <= TOL
    assert O.max_rel_err(_np(du), ru) <= TOL


def test_layer_ops_reject_bad_input():
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    x = torch.zeros(4, 12, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(_lib.LobraError):
        _lib.lobra_rmsnorm_fwd(x, x[0], 1e-5, x, torch.zeros(4, device="cuda"))   # h % 8 != 0
    cu = torch.tensor([0, 4], dtype=torch.int32, device="cuda")
    with pytest.raises(_lib.LobraError):
        _lib.lobra_rope(cu, 4, 1, 12, 10000.0, x)                                   # head_dim % 16
