"""Out-of-bounds write checks of our own (compute-sanitizer is not available on the GPU pool).

Every device buffer a C-ABI call writes (outputs, saved activations, workspaces) is placed
inside a larger allocation with 64 KiB guard bands on both sides.  Everything starts as
0xFF bytes, which is NaN for bf16 and fp32.  After the call:
  * both guard bands still hold 0xFF (no write outside the buffer the caller passed);
  * outputs the call fully defines contain no NaN (every element was written);
  * the results equal, bit for bit, a second run on ordinarily allocated buffers.
The shapes are ragged on purpose: tails in T, in/out not multiples of 128 / 256, ranks 8-64,
tasks interleaved, a task without tokens, attention lengths off the 128-row tile.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GUARD = 65536


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


class Guarded:
    def __init__(self, torch, shape, dtype, nbytes=None):
        self.torch = torch
        el = torch.empty(0, dtype=dtype).element_size()
        n = int(np.prod(shape)) * el if nbytes is None else int(nbytes)
        self.n = n
        pad = (n + 1023) // 1024 * 1024
        self.raw = torch.full((GUARD + pad + GUARD,), 0xFF, dtype=torch.uint8, device="cuda")
        self.t = self.raw[GUARD:GUARD + n].view(dtype)
        if nbytes is None:
            self.t = self.t.view(*shape)

    def guards_intact(self):
        return bool((self.raw[:GUARD] == 0xFF).all()) and bool((self.raw[GUARD + self.n:] == 0xFF).all())


def _check(bufs, defined):
    for name, g in bufs.items():
        assert g.guards_intact(), f"{name}: write outside the buffer"
    for name in defined:
        assert not bool(bufs[name].t.isnan().any()), f"{name}: elements left unwritten"


def _lora_case(torch, seed=0):
    rng = np.random.default_rng(seed)
    lens = np.array([1, 130, 77, 0, 300, 45, 129, 256, 3], np.int32)
    tasks = np.array([0, 2, 1, 3, 2, 0, 4, 1, 2], np.int32)
    ranks = np.array([16, 8, 64, 32, 24], np.int32)   # task 3 only has an empty sequence
    scales = np.array([2.0, 0.5, 1.0, 1.5, 0.25], np.float32)
    return lens, tasks, ranks, scales, int(lens.sum())


@pytest.mark.parametrize("dtype_name,d_in,d_out", [("bf16", 320, 448), ("bf16", 4096, 704), ("fp32", 96, 80)])
def test_lora_fwd_bwd_stays_in_bounds(dtype_name, d_in, d_out):
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    td = torch.bfloat16 if dtype_name == "bf16" else torch.float32
    code = _lib.LOBRA_BF16 if dtype_name == "bf16" else _lib.LOBRA_FP32
    lens, tasks, ranks, scales, T = _lora_case(torch)
    R = int(ranks.sum())
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    rn = lambda *s: (torch.randn(*s, generator=g, device="cuda") * 0.5).to(td)
    X, W, A, B, dY = rn(T, d_in), rn(d_out, d_in), rn(R, d_in), rn(d_out, R), rn(T, d_out)
    ws_n = _lib.lobra_lora_workspace_bytes(code, d_in, d_out, lens, tasks, ranks, scales)
    hs_n = _lib.lobra_lora_saved_bytes(code, d_in, d_out, lens, tasks, ranks, scales)

    def run(alloc):
        b = {"Y": alloc((T, d_out), td), "Hs": alloc(None, torch.uint8, hs_n), "ws": alloc(None, torch.uint8, ws_n),
             "dX": alloc((T, d_in), td), "dA": alloc((R, d_in), torch.float32),
             "dB": alloc((d_out, R), torch.float32)}
        t = {k: v.t if isinstance(v, Guarded) else v for k, v in b.items()}
        _lib.lobra_lora_fwd(X, W, A, B, ranks, scales, lens, tasks, t["Y"], t["Hs"], t["ws"])
        _lib.lobra_lora_bwd(X, W, A, B, ranks, scales, lens, tasks, t["Hs"], dY, t["dX"], t["dA"], t["dB"], t["ws"])
        torch.cuda.synchronize()
        return b, t

    guarded, gt = run(lambda s, dt, n=None: Guarded(torch, s, dt, n))
    _check(guarded, ["Y", "dX", "dA", "dB"])
    _, plain = run(lambda s, dt, n=None: torch.empty(s if n is None else (n,), dtype=dt, device="cuda"))
    for k in ("Y", "dX", "dA", "dB"):
        assert torch.equal(gt[k], plain[k]), k


@pytest.mark.parametrize("d_in,outs,ranks", [(512, [512, 192, 192], [16, 8, 64, 32, 24]),
                                              (448, [704, 704], [64, 64, 8, 16, 32])])
def test_group_fwd_bwd_stays_in_bounds(d_in, outs, ranks):
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    td, code = torch.bfloat16, _lib.LOBRA_BF16
    lens, tasks, _, scales, T = _lora_case(torch, 1)
    ranks = np.array(ranks, np.int32)
    R = int(ranks.sum())
    g = torch.Generator(device="cuda")
    g.manual_seed(2)
    rn = lambda *s: (torch.randn(*s, generator=g, device="cuda") * 0.5).to(td)
    X = rn(T, d_in)
    Ws = [rn(o, d_in) for o in outs]
    As = [rn(R, d_in) for _ in outs]
    Bs = [rn(o, R) for o in outs]
    dYs = [rn(T, o) for o in outs]
    ws_n = _lib.lobra_lora_group_workspace_bytes(code, d_in, outs, lens, tasks, ranks, scales)
    hs_n = _lib.lobra_lora_group_saved_bytes(code, d_in, outs, lens, tasks, ranks, scales)

    def run(alloc):
        b = {"Hs": alloc(None, torch.uint8, hs_n), "ws": alloc(None, torch.uint8, ws_n), "dX": alloc((T, d_in), td)}
        for p, o in enumerate(outs):
            b[f"Y{p}"] = alloc((T, o), td)
            b[f"dA{p}"] = alloc((R, d_in), torch.float32)
            b[f"dB{p}"] = alloc((o, R), torch.float32)
        t = {k: v.t if isinstance(v, Guarded) else v for k, v in b.items()}
        n = len(outs)
        _lib.lobra_lora_group_fwd(X, Ws, As, Bs, ranks, scales, lens, tasks, [t[f"Y{p}"] for p in range(n)],
                                  t["Hs"], t["ws"])
        _lib.lobra_lora_group_bwd(X, Ws, As, Bs, ranks, scales, lens, tasks, t["Hs"], dYs, t["dX"],
                                  [t[f"dA{p}"] for p in range(n)], [t[f"dB{p}"] for p in range(n)], t["ws"])
        torch.cuda.synchronize()
        return b, t

    guarded, gt = run(lambda s, dt, n=None: Guarded(torch, s, dt, n))
    defined = ["dX"] + [f"{k}{p}" for p in range(len(outs)) for k in ("Y", "dA", "dB")]
    _check(guarded, defined)
    _, plain = run(lambda s, dt, n=None: torch.empty(s if n is None else (n,), dtype=dt, device="cuda"))
    for k in defined:
        assert torch.equal(gt[k], plain[k]), k


@pytest.mark.parametrize("lens,H,Hkv", [([1, 300, 57, 129, 200, 33], 4, 2), ([384, 5, 250], 2, 1)])
def test_attention_fwd_bwd_stays_in_bounds(lens, H, Hkv):
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    T = sum(lens)
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    rn = lambda *s: torch.randn(*s, generator=g, device="cuda").to(torch.bfloat16)
    q, k, v, dO = rn(T, H, 128), rn(T, Hkv, 128), rn(T, Hkv, 128), rn(T, H, 128)
    wsf = _lib.lobra_attn_workspace_bytes(lens, H)
    wsb = _lib.lobra_attn_bwd_workspace_bytes(lens, H, Hkv)

    def run(alloc):
        b = {"O": alloc((T, H, 128), torch.bfloat16), "lse": alloc((H, T), torch.float32),
             "wsf": alloc(None, torch.uint8, wsf), "wsb": alloc(None, torch.uint8, wsb),
             "dQ": alloc((T, H, 128), torch.bfloat16), "dK": alloc((T, Hkv, 128), torch.bfloat16),
             "dV": alloc((T, Hkv, 128), torch.bfloat16)}
        t = {k_: v_.t if isinstance(v_, Guarded) else v_ for k_, v_ in b.items()}
        _lib.lobra_attn_fwd(lens, q, k, v, t["O"], t["lse"], t["wsf"])
        _lib.lobra_attn_bwd(lens, q, k, v, t["O"], dO, t["lse"], t["dQ"], t["dK"], t["dV"], t["wsb"])
        torch.cuda.synchronize()
        return b, t

    guarded, gt = run(lambda s, dt, n=None: Guarded(torch, s, dt, n))
    defined = ["O", "lse", "dQ", "dK", "dV"]
    _check(guarded, defined)
    _, plain = run(lambda s, dt, n=None: torch.empty(s if n is None else (n,), dtype=dt, device="cuda"))
    for k_ in defined:
        assert torch.equal(gt[k_], plain[k_]), k_


def test_layer_ops_stay_in_bounds():
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    T, h = 333, 4096
    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    rn = lambda *s: torch.randn(*s, generator=g, device="cuda").to(torch.bfloat16)
    X, Rr, gam, dY, dRes = rn(T, h), rn(T, h), rn(h), rn(T, h), rn(T, h)
    b = {"Y": Guarded(torch, (T, h), torch.bfloat16), "rstd": Guarded(torch, (T,), torch.float32),
         "S": Guarded(torch, (T, h), torch.bfloat16), "dS": Guarded(torch, (T, h), torch.bfloat16),
         "act": Guarded(torch, (T, h), torch.bfloat16),
         "dg": Guarded(torch, (T, h), torch.bfloat16), "du": Guarded(torch, (T, h), torch.bfloat16)}
    t = {k: v.t for k, v in b.items()}
    _lib.lobra_rmsnorm_fwd(X, gam, 1e-5, t["Y"], t["rstd"], R=Rr, S_out=t["S"])
    _lib.lobra_rmsnorm_bwd(dY, t["S"], gam, t["rstd"], t["dS"], dRes=dRes)
    _lib.lobra_swiglu_fwd(X, Rr, t["act"])
    _lib.lobra_swiglu_bwd(dY, X, Rr, t["dg"], t["du"])
    torch.cuda.synchronize()
    _check(b, list(b))
