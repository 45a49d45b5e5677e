"""GPU: projection groups (SURVEY §8(a) a1 "inputs sharing X are done in one pass") through
the C ABI.  A group call must give BITWISE the results of the equivalent sequence of
single-projection calls (the banded shrink / dA reduction compute every output column with
the same MMAs in the same order), and match the fp64 oracle per projection at the bf16
tolerance.  Also the fallback (bands do not fit: num_proj * qp > 64), the 70B-style group
with unequal widths (q 8192 / k,v 1024), accumulation, and the empty batch.
"""
import numpy as np
import pytest

from oracle import lora as O
from workloads import synth

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _workload(seed, ranks, scales, n, lmax):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, lmax, size=n).astype(np.int32)
    tids = rng.integers(0, len(ranks), size=n).astype(np.int32)
    o = np.argsort(tids, kind="stable")
    tasks = [synth.TaskSpec(f"t{i}", 0, 0, 1, r, s) for i, (r, s) in enumerate(zip(ranks, scales))]
    return synth.Workload("grp", tasks, lens[o], tids[o], lmax)


def _tensors(wl, d_in, outs, seed):
    """Per projection: W_p, A_p, B_p, dY_p (seeded); shared X."""
    ts = [synth.layer_tensors(wl, d_in, o, seed=seed + 7 * p) for p, o in enumerate(outs)]
    X = ts[0]["X"]
    return X, ts


def _run(wl, d_in, outs, seed, group=True, accumulate=False):
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    dev = torch.device("cuda:0")
    up = lambda a: torch.from_numpy(np.ascontiguousarray(synth.round_bf16(a))).to(dev).to(torch.bfloat16)
    X, ts = _tensors(wl, d_in, outs, seed)
    Xd = up(X)
    Ws = [up(t["W"]) for t in ts]
    As = [up(t["A"]) for t in ts]
    Bs = [up(t["B"]) for t in ts]
    dYs = [up(t["dY"]) for t in ts]
    T, Rs = wl.T, int(wl.ranks.sum())
    r, s, L, K = wl.ranks, wl.scales, wl.seq_lens, wl.seq_task
    rng = np.random.default_rng(seed + 99)
    init_dX = up(rng.standard_normal((T, d_in))) if accumulate else None
    init_dA = [torch.from_numpy(rng.standard_normal((Rs, d_in)).astype(np.float32)).to(dev) for _ in outs]
    init_dB = [torch.from_numpy(rng.standard_normal((o, Rs)).astype(np.float32)).to(dev) for o in outs]
    if accumulate:
        dX = init_dX.clone()
        dA = [a.clone() for a in init_dA]
        dB = [b.clone() for b in init_dB]
    else:
        dX = torch.full((T, d_in), float("nan"), device=dev, dtype=torch.bfloat16)
        dA = [torch.full((Rs, d_in), float("nan"), device=dev) for _ in outs]
        dB = [torch.full((o, Rs), float("nan"), device=dev) for o in outs]
    Ys = [torch.full((T, o), float("nan"), device=dev, dtype=torch.bfloat16) for o in outs]
    if group:
        ws = torch.empty(_lib.lobra_lora_group_workspace_bytes(_lib.LOBRA_BF16, d_in, outs, L, K, r, s),
                         device=dev, dtype=torch.uint8)
        Hs = torch.empty(_lib.lobra_lora_group_saved_bytes(_lib.LOBRA_BF16, d_in, outs, L, K, r, s),
                         device=dev, dtype=torch.uint8)
        _lib.lobra_lora_group_fwd(Xd, Ws, As, Bs, r, s, L, K, Ys, Hs, ws)
        _lib.lobra_lora_group_bwd(Xd, Ws, As, Bs, r, s, L, K, Hs, dYs, dX, dA, dB, ws,
                                  accumulate_dx=accumulate, accumulate_dadb=accumulate)
    else:
        for p, o in enumerate(outs):
            ws = torch.empty(_lib.lobra_lora_workspace_bytes(_lib.LOBRA_BF16, d_in, o, L, K, r, s),
                             device=dev, dtype=torch.uint8)
            Hs = torch.empty(_lib.lobra_lora_saved_bytes(_lib.LOBRA_BF16, d_in, o, L, K, r, s),
                             device=dev, dtype=torch.uint8)
            _lib.lobra_lora_fwd(Xd, Ws[p], As[p], Bs[p], r, s, L, K, Ys[p], Hs, ws)
            _lib.lobra_lora_bwd(Xd, Ws[p], As[p], Bs[p], r, s, L, K, Hs, dYs[p], dX, dA[p], dB[p], ws,
                                accumulate_dx=accumulate or p > 0, accumulate_dadb=accumulate)
    torch.cuda.synchronize()
    f = lambda x: x.float().cpu().numpy().astype(np.float64)
    res = {"Y": [f(y) for y in Ys], "dX": f(dX), "dA": [f(a) for a in dA], "dB": [f(b) for b in dB]}
    init = None
    if accumulate:
        init = {"dX": f(init_dX), "dA": [f(a) for a in init_dA], "dB": [f(b) for b in init_dB]}
    return res, X, ts, init


def _oracle_check(wl, X, ts, res, init=None):
    b = lambda a: synth.round_bf16(a).astype(np.float64)
    Xo = b(X)
    dX_sum = np.zeros_like(res["dX"]) if init is None else init["dX"].copy()
    errs = {}
    for p, t in enumerate(ts):
        args = (Xo, b(t["W"]), b(t["A"]), b(t["B"]), wl.ranks.tolist(), wl.scales, wl.seq_lens, wl.seq_task)
        Yo = O.lora_fwd(*args)
        dXo, dAo, dBo = O.lora_bwd(*args, b(t["dY"]))
        dX_sum += dXo
        if init is not None:
            dAo = dAo + init["dA"][p]
            dBo = dBo + init["dB"][p]
        errs[f"Y{p}"] = O.max_rel_err(res["Y"][p], Yo)
        errs[f"dA{p}"] = O.max_rel_err(res["dA"][p], dAo)
        errs[f"dB{p}"] = O.max_rel_err(res["dB"][p], dBo)
    errs["dX"] = O.max_rel_err(res["dX"], dX_sum)
    bad = {k: v for k, v in errs.items() if not (v <= BF16_TOL)}
    assert not bad, f"tolerance exceeded: {bad} (all: {errs})"


def _same(a, b):
    for k in ("Y", "dA", "dB"):
        for p, (x, y) in enumerate(zip(a[k], b[k])):
            assert np.array_equal(x, y), f"{k}[{p}] differs: max |d| = {np.nanmax(np.abs(x - y))}"
    assert np.array_equal(a["dX"], b["dX"]), "dX differs"


@pytest.mark.parametrize("np_,ranks", [(3, (16, 16, 8)), (2, (32, 16, 24)), (4, (16, 8, 16))])
def test_group_equals_single_sequence_bitwise(np_, ranks):
    """qkv-like (3 x 16 bands), gate/up-like (2 x 32 bands), 4 projections of 16; mixed
    task tiles, ragged tail, ranks not multiples of 16 (padded bands), odd T."""
    wl = _workload(3 + np_, ranks, (2.0, 0.5, 1.0), 11, 300)
    d_in = 320
    outs = [384, 256, 512, 128][:np_]
    g, X, ts, _ = _run(wl, d_in, outs, seed=21)
    s, _, _, _ = _run(wl, d_in, outs, seed=21, group=False)
    _same(g, s)
    _oracle_check(wl, X, ts, g)


def test_group_accumulate():
    wl = _workload(8, (16, 16), (1.0, 4.0), 7, 200)
    d_in, outs = 256, [256, 384, 128]
    g, X, ts, init = _run(wl, d_in, outs, seed=5, accumulate=True)
    s, _, _, _ = _run(wl, d_in, outs, seed=5, group=False, accumulate=True)
    _same(g, s)
    _oracle_check(wl, X, ts, g, init)


def test_group_fallback_when_bands_do_not_fit():
    """3 x qp(64) > 64: the call runs the single-projection sequence internally."""
    wl = _workload(9, (64, 16, 33), (1.0, 2.0, 0.5), 8, 220)
    d_in, outs = 192, [256, 128, 256]
    g, X, ts, _ = _run(wl, d_in, outs, seed=8)
    s, _, _, _ = _run(wl, d_in, outs, seed=8, group=False)
    _same(g, s)
    _oracle_check(wl, X, ts, g)


def test_group_70b_qkv_shapes():
    """70B GQA q / k / v widths (8192 / 1024 / 1024) sharing X (in = 8192), C2-like mix of
    4 tasks r = 16, ~2.3K tokens; sampled against the oracle (full check is too slow)."""
    tasks = synth.c2_tasks()
    wl = synth.pack_tokens(tasks, 2304, 1024, seed=4, name="g70")
    d_in, outs = 8192, [8192, 1024, 1024]
    g, X, ts, _ = _run(wl, d_in, outs, seed=2)
    s, _, _, _ = _run(wl, d_in, outs, seed=2, group=False)
    _same(g, s)


def test_group_empty_batch_zeroes_grads():
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    dev = torch.device("cuda:0")
    r, s = [16, 8], [1.0, 1.0]
    L, K = [0, 0], [0, 1]
    outs, d_in = [128, 256], 128
    ws = torch.empty(max(256, _lib.lobra_lora_group_workspace_bytes(_lib.LOBRA_BF16, d_in, outs, L, K, r, s)),
                     device=dev, dtype=torch.uint8)
    Hs = torch.empty(_lib.lobra_lora_group_saved_bytes(_lib.LOBRA_BF16, d_in, outs, L, K, r, s), device=dev,
                     dtype=torch.uint8)
    X = torch.zeros(1, d_in, device=dev, dtype=torch.bfloat16)   # non-null dummies (T = 0)
    Ws = [torch.zeros(o, d_in, device=dev, dtype=torch.bfloat16) for o in outs]
    As = [torch.zeros(24, d_in, device=dev, dtype=torch.bfloat16) for _ in outs]
    Bs = [torch.zeros(o, 24, device=dev, dtype=torch.bfloat16) for o in outs]
    Ys = [torch.zeros(1, o, device=dev, dtype=torch.bfloat16) for o in outs]
    dYs = [torch.zeros(1, o, device=dev, dtype=torch.bfloat16) for o in outs]
    dA = [torch.full((24, d_in), 3.0, device=dev) for _ in outs]
    dB = [torch.full((o, 24), 3.0, device=dev) for o in outs]
    dX = torch.zeros(1, d_in, device=dev, dtype=torch.bfloat16)
    _lib.lobra_lora_group_fwd(X, Ws, As, Bs, r, s, L, K, Ys, Hs, ws)
    _lib.lobra_lora_group_bwd(X, Ws, As, Bs, r, s, L, K, Hs, dYs, dX, dA, dB, ws)
    torch.cuda.synchronize()
    for a, b in zip(dA, dB):
        assert not a.any() and not b.any()
    for a in dA:
        a.fill_(3.0)
    _lib.lobra_lora_group_bwd(X, Ws, As, Bs, r, s, L, K, Hs, dYs, dX, dA, dB, ws, accumulate_dadb=True)
    torch.cuda.synchronize()
    assert all((a == 3.0).all() for a in dA)


def test_group_errors():
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    with pytest.raises(_lib.LobraError):     # out not a multiple of 64
        _lib.lobra_lora_group_workspace_bytes(_lib.LOBRA_BF16, 128, [128, 100], [5], [0], [8], [1.0])
    with pytest.raises(_lib.LobraError):     # more than 4 projections
        _lib.lobra_lora_group_workspace_bytes(_lib.LOBRA_BF16, 128, [128] * 5, [5], [0], [8], [1.0])


def test_layer_grouped_equals_ungrouped():
    """LoraLayer drives q/k/v and gate/up through the group calls: the outputs, dX and the
    flat adapter-gradient buffer are bitwise those of the per-projection calls."""
    torch = _torch()
    from paper_2509_01193_b200.layer import LoraLayer
    shapes = [("q", 256, 256, "col", "attn"), ("k", 256, 128, "col", "attn"), ("v", 256, 128, "col", "attn"),
              ("o", 256, 256, "row", "o_in"), ("gate", 256, 512, "col", "mlp"), ("up", 256, 512, "col", "mlp"),
              ("down", 512, 256, "row", "down_in")]
    wl = _workload(12, (16, 8, 16), (2.0, 1.0, 0.5), 9, 200)
    out = []
    for grouped in (True, False):
        layer = LoraLayer(shapes, wl.ranks, wl.scales, "cuda:0", seed=3, group_inputs=grouped)
        io = layer.alloc_io(wl.T, seed=4)
        for acc in (False, True):
            layer.forward(wl.seq_lens, wl.seq_task, io, wl.T)
            layer.backward(wl.seq_lens, wl.seq_task, io, wl.T, accumulate_dadb=acc)
        torch.cuda.synchronize()
        out.append(({k: v.clone() for k, v in io["Y"].items()}, {k: v.clone() for k, v in io["dX"].items()},
                    layer.flat_grad.clone()))
    (Yg, dXg, fg), (Yu, dXu, fu) = out
    for k in Yg:
        assert torch.equal(Yg[k], Yu[k]), k
    for k in dXg:
        assert torch.equal(dXg[k], dXu[k]), k
    assert torch.equal(fg, fu)
    assert torch.isfinite(fg).all()


def test_group_c2_qkv_full_size_equals_single_sequence():
    """BASELINE config 2 at full size (T = 16384, 4 tasks r = 16, s = 2; 7B q/k/v 4096 ->
    4096 sharing X), in the launch configuration bench.py times: the group call gives
    bitwise the single-projection sequence (which test_gpu_lora checks against the oracle
    at this size)."""
    wl = synth.config_c2()
    d_in, outs = 4096, [4096, 4096, 4096]
    g, _, _, _ = _run(wl, d_in, outs, seed=31)
    s, _, _, _ = _run(wl, d_in, outs, seed=31, group=False)
    _same(g, s)
    for y in g["Y"]:
        assert np.isfinite(y).all()


def test_group_many_tasks_full_batch():
    """128 tiles holding 24 interleaved tasks (k_shrink per tile with several passes, many dY
    segments), unequal widths (q 192 / k,v 64): group == single-projection calls bitwise."""
    rng = np.random.default_rng(9)
    lens = []
    while sum(lens) < 16384:
        lens.append(int(rng.integers(5, 90)))
    lens[-1] -= sum(lens) - 16384
    G = 24
    ts = [synth.TaskSpec(f"t{i}", 0, 0, 1, 16, 0.5 + 0.5 * (i % 4)) for i in range(G)]
    wl = synth.Workload("mix24", ts, np.array(lens, np.int32),
                        np.array([(i * 7) % G for i in range(len(lens))], np.int32), 0)
    g, X, ts_, _ = _run(wl, 256, [192, 64, 64], seed=3)
    s, _, _, _ = _run(wl, 256, [192, 64, 64], seed=3, group=False)
    _same(g, s)


def test_wide_group_planes_full_batch():
    """A group whose bands exceed the 64-wide slot (3 x rank 64 = 192 columns, C3's q/k/v):
    one k_shrink pass over X writes every projection's H_s plane (112 tiles, mixed ranks
    8-64, ragged last tile); results bitwise those of the single-projection calls."""
    rng = np.random.default_rng(12)
    lens = []
    while sum(lens) < 14300:
        lens.append(int(rng.integers(20, 400)))
    lens[-1] -= sum(lens) - 14300
    ranks = [8, 16, 32, 64] * 2
    ts = [synth.TaskSpec(f"t{i}", 0, 0, 1, r, 0.5 + 0.5 * (i % 4)) for i, r in enumerate(ranks)]
    wl = synth.Workload("wide", ts, np.array(lens, np.int32),
                        np.array(sorted(i % 8 for i in range(len(lens))), np.int32), 0)
    g, X, ts_, _ = _run(wl, 256, [192, 64, 64], seed=4)
    s, _, _, _ = _run(wl, 256, [192, 64, 64], seed=4, group=False)
    _same(g, s)


def test_wide_group_c3_full_size_bitwise():
    """BASELINE config 3 at full size in the bench launch configuration: q/k/v (4096 -> 4096)
    over the C3 batch (16 tasks, ranks 8-64: a wide group, planes shrink, 512 tiles), device
    tensors; group == single-projection calls bit for bit (the single path is checked against
    the oracle at this size in test_gpu_lora.test_bf16_c3_q_projection_full_size)."""
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    dev = torch.device("cuda:0")
    wl = synth.config_c3()
    T, d_in, outs = wl.T, 4096, [4096, 4096, 4096]
    r, s, L, K = wl.ranks, wl.scales, wl.seq_lens, wl.seq_task
    Rs = int(r.sum())
    g = torch.Generator(device=dev).manual_seed(5)
    rn = lambda *sh, sc=1.0: (torch.randn(*sh, generator=g, device=dev) * sc).to(torch.bfloat16)
    X = rn(T, d_in)
    Ws = [rn(o, d_in, sc=d_in ** -0.5) for o in outs]
    As = [rn(Rs, d_in, sc=d_in ** -0.5) for _ in outs]
    Bs = [rn(o, Rs, sc=0.125) for o in outs]
    dYs = [rn(T, o) for o in outs]

    def run(group):
        Ys = [torch.empty(T, o, device=dev, dtype=torch.bfloat16) for o in outs]
        dX = torch.empty(T, d_in, device=dev, dtype=torch.bfloat16)
        dA = [torch.empty(Rs, d_in, device=dev) for _ in outs]
        dB = [torch.empty(o, Rs, device=dev) for o in outs]
        if group:
            ws = torch.empty(_lib.lobra_lora_group_workspace_bytes(_lib.LOBRA_BF16, d_in, outs, L, K, r, s),
                             device=dev, dtype=torch.uint8)
            Hs = torch.empty(_lib.lobra_lora_group_saved_bytes(_lib.LOBRA_BF16, d_in, outs, L, K, r, s),
                             device=dev, dtype=torch.uint8)
            _lib.lobra_lora_group_fwd(X, Ws, As, Bs, r, s, L, K, Ys, Hs, ws)
            _lib.lobra_lora_group_bwd(X, Ws, As, Bs, r, s, L, K, Hs, dYs, dX, dA, dB, ws)
        else:
            for p, o in enumerate(outs):
                ws = torch.empty(_lib.lobra_lora_workspace_bytes(_lib.LOBRA_BF16, d_in, o, L, K, r, s),
                                 device=dev, dtype=torch.uint8)
                Hs = torch.empty(_lib.lobra_lora_saved_bytes(_lib.LOBRA_BF16, d_in, o, L, K, r, s),
                                 device=dev, dtype=torch.uint8)
                _lib.lobra_lora_fwd(X, Ws[p], As[p], Bs[p], r, s, L, K, Ys[p], Hs, ws)
                _lib.lobra_lora_bwd(X, Ws[p], As[p], Bs[p], r, s, L, K, Hs, dYs[p], dX, dA[p], dB[p], ws,
                                    accumulate_dx=p > 0)
        torch.cuda.synchronize()
        return Ys, dX, dA, dB

    a, b = run(True), run(False)
    for p in range(3):
        assert torch.equal(a[0][p], b[0][p]), f"Y[{p}]"
        assert torch.equal(a[2][p], b[2][p]), f"dA[{p}]"
        assert torch.equal(a[3][p], b[3][p]), f"dB[{p}]"
    assert torch.equal(a[1], b[1]), "dX"
