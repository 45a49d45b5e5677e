"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle (run under gpurun).

Tolerances (BASELINE.json north_star): bf16 inputs with fp32 accumulation, max relative
error 2e-2; fp32 path 1e-5.  Error metric per output tensor (reading Q9):
max|gpu - oracle| / max|oracle|; dA_t and dB_t per task.
"""
import numpy as np
import pytest

from oracle import lora as O
from workloads import synth

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2
FP32_TOL = 1e-5


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def run_lib(dtype, wl, t, d_in, d_out, accumulate_dx=False, accumulate_dadb=False, init=None):
    """Runs fwd + bwd through the C ABI; returns host fp64 arrays (Y, dX, dA, dB, Hs)."""
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    dev = torch.device("cuda:0")
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    code = _lib.LOBRA_BF16 if dtype == "bf16" else _lib.LOBRA_FP32

    def up(a):
        a = synth.round_bf16(a) if dtype == "bf16" else np.asarray(a, np.float32)
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(td)

    X, W, A, B, dY = (up(t[k]) for k in ("X", "W", "A", "B", "dY"))
    T = wl.T
    ranks, scales = wl.ranks, wl.scales
    Y = torch.empty(T, d_out, device=dev, dtype=td)
    ws_n = _lib.lobra_lora_workspace_bytes(code, d_in, d_out, wl.seq_lens, wl.seq_task, ranks, scales)
    hs_n = _lib.lobra_lora_saved_bytes(code, d_in, d_out, wl.seq_lens, wl.seq_task, ranks, scales)
    ws = torch.empty(ws_n, device=dev, dtype=torch.uint8)
    Hs = torch.empty(hs_n, device=dev, dtype=torch.uint8)
    _lib.lobra_lora_fwd(X, W, A, B, ranks, scales, wl.seq_lens, wl.seq_task, Y, Hs, ws)
    Rs = int(ranks.sum())
    if init is not None:
        dX = up(init["dX"])
        dA = torch.from_numpy(init["dA"].astype(np.float32)).to(dev)
        dB = torch.from_numpy(init["dB"].astype(np.float32)).to(dev)
    else:
        dX = torch.full((T, d_in), float("nan"), device=dev, dtype=td)
        dA = torch.full((Rs, d_in), float("nan"), device=dev, dtype=torch.float32)
        dB = torch.full((d_out, Rs), float("nan"), device=dev, dtype=torch.float32)
    _lib.lobra_lora_bwd(X, W, A, B, ranks, scales, wl.seq_lens, wl.seq_task, Hs, dY, dX, dA, dB, ws,
                        accumulate_dx=accumulate_dx, accumulate_dadb=accumulate_dadb)
    torch.cuda.synchronize()
    f = lambda x: x.float().cpu().numpy().astype(np.float64)
    return f(Y), f(dX), f(dA), f(dB), Hs


def oracle_inputs(dtype, t):
    conv = (lambda a: synth.round_bf16(a).astype(np.float64)) if dtype == "bf16" else \
        (lambda a: np.asarray(a, np.float32).astype(np.float64))
    return {k: conv(v) for k, v in t.items()}


def check_all(wl, t, got, tol, d_in, d_out):
    Y, dX, dA, dB = got[:4]
    args = (t["X"], t["W"], t["A"], t["B"], wl.ranks.tolist(), wl.scales, wl.seq_lens, wl.seq_task)
    Yo = O.lora_fwd(*args)
    dXo, dAo, dBo = O.lora_bwd(*args, t["dY"])
    errs = {"Y": O.max_rel_err(Y, Yo), "dX": O.max_rel_err(dX, dXo)}
    roff = np.concatenate([[0], np.cumsum(wl.ranks)])
    present = set(wl.seq_task[wl.seq_lens > 0].tolist())
    for k in range(len(wl.ranks)):
        a, b = roff[k], roff[k + 1]
        if k in present:
            errs[f"dA{k}"] = O.max_rel_err(dA[a:b], dAo[a:b])
            errs[f"dB{k}"] = O.max_rel_err(dB[:, a:b], dBo[:, a:b])
        else:   # reading Q10: no tokens -> exact zeros when overwriting
            assert not dA[a:b].any() and not dB[:, a:b].any()
    bad = {k: v for k, v in errs.items() if not (v <= tol)}
    assert not bad, f"tolerance {tol} exceeded: {bad} (all: {errs})"
    return errs


def test_c1_fp32():
    """BASELINE config 1: tiny 64x64, 2 tasks r=4, 8 sequences of 3-40 tokens, fp32."""
    wl = synth.config_c1()
    t = synth.layer_tensors(wl, 64, 64, seed=1)
    got = run_lib("fp32", wl, t, 64, 64)
    check_all(wl, oracle_inputs("fp32", t), got, FP32_TOL, 64, 64)


def _medium(seed=5, ranks=(8, 16, 64), scales=(2.0, 0.5, 1.0), n=9, lmax=160, group=True,
            used=None):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, lmax, size=n).astype(np.int32)
    tids = rng.integers(0, len(ranks) if used is None else used, size=n).astype(np.int32)
    if group:
        o = np.argsort(tids, kind="stable")
        lens, tids = lens[o], tids[o]
    tasks = [synth.TaskSpec(f"t{i}", 0, 0, 1, r, s) for i, (r, s) in enumerate(zip(ranks, scales))]
    return synth.Workload("medium", tasks, lens, tids, lmax)


@pytest.mark.parametrize("group", [True, False])
def test_bf16_medium(group):
    """Several M tiles with a ragged tail, mixed-task tiles, 3 tasks of ranks 8/16/64,
    N = 384 (one full 256-wide tile + a 128 tail)."""
    wl = _medium(group=group)
    d_in, d_out = 256, 384
    t = synth.layer_tensors(wl, d_in, d_out, seed=11)
    got = run_lib("bf16", wl, t, d_in, d_out)
    check_all(wl, oracle_inputs("bf16", t), got, BF16_TOL, d_in, d_out)


def test_bf16_fp32_paths_agree_medium():
    wl = _medium(seed=6)
    t = synth.layer_tensors(wl, 128, 192, seed=12)
    check_all(wl, oracle_inputs("fp32", t), run_lib("fp32", wl, t, 128, 192), FP32_TOL, 128, 192)


def test_bf16_W_zero_isolates_adapters():
    wl = _medium(seed=7)
    t = synth.layer_tensors(wl, 192, 256, seed=13, zero_W=True)
    check_all(wl, oracle_inputs("bf16", t), run_lib("bf16", wl, t, 192, 256), BF16_TOL, 192, 256)


def test_bf16_B_zero_bitwise_equals_scale_zero():
    """B_t = 0 adds exact zeros to the fp32 accumulator: Y(B=0) == Y(s=0) bit for bit,
    and both match the base X W^T."""
    wl = _medium(seed=8)
    t = synth.layer_tensors(wl, 128, 256, seed=14, zero_B=True)
    Y0 = run_lib("bf16", wl, t, 128, 256)[0]
    wl2 = _medium(seed=8, scales=(0.0, 0.0, 0.0))
    t2 = synth.layer_tensors(wl2, 128, 256, seed=14)
    Y1 = run_lib("bf16", wl2, t2, 128, 256)[0]
    assert np.array_equal(Y0, Y1)
    ti = oracle_inputs("bf16", t)
    assert O.max_rel_err(Y0, ti["X"] @ ti["W"].T) < BF16_TOL


def test_bf16_packing_order_rows_bitwise():
    """Per-sequence Y rows do not depend on where the sequence is packed."""
    wl = _medium(seed=9, n=7)
    d_in, d_out = 128, 256
    t = synth.layer_tensors(wl, d_in, d_out, seed=15)
    Y = run_lib("bf16", wl, t, d_in, d_out)[0]
    perm = np.array([3, 6, 0, 5, 1, 4, 2])
    offs = np.concatenate([[0], np.cumsum(wl.seq_lens)])
    rows = np.concatenate([np.arange(offs[k], offs[k + 1]) for k in perm]).astype(np.int64)
    wl2 = synth.Workload("perm", wl.tasks, wl.seq_lens[perm], wl.seq_task[perm], wl.l_max)
    t2 = dict(t)
    t2["X"], t2["dY"] = t["X"][rows], t["dY"][rows]
    Y2 = run_lib("bf16", wl2, t2, d_in, d_out)[0]
    assert np.array_equal(Y[rows], Y2)


def test_bf16_accumulate_flags():
    """accumulate_dx / accumulate_dadb add to the existing buffers (gradient
    accumulation)."""
    wl = _medium(seed=10)
    d_in, d_out = 128, 192
    t = synth.layer_tensors(wl, d_in, d_out, seed=16)
    rng = np.random.default_rng(0)
    Rs = int(wl.ranks.sum())
    init = {"dX": rng.standard_normal((wl.T, d_in)).astype(np.float32),
            "dA": rng.standard_normal((Rs, d_in)), "dB": rng.standard_normal((d_out, Rs))}
    got = run_lib("bf16", wl, t, d_in, d_out, accumulate_dx=True, accumulate_dadb=True, init=init)
    ti = oracle_inputs("bf16", t)
    args = (ti["X"], ti["W"], ti["A"], ti["B"], wl.ranks.tolist(), wl.scales, wl.seq_lens, wl.seq_task)
    dXo, dAo, dBo = O.lora_bwd(*args, ti["dY"])
    assert O.max_rel_err(got[1], dXo + synth.round_bf16(init["dX"])) < BF16_TOL
    assert O.max_rel_err(got[2], dAo + init["dA"].astype(np.float32)) < BF16_TOL
    assert O.max_rel_err(got[3], dBo + init["dB"].astype(np.float32)) < BF16_TOL


def test_bf16_task_without_tokens_gets_zero_grads():
    wl = _medium(seed=11, ranks=(8, 16, 64, 32), scales=(1.0, 1.0, 1.0, 3.0), used=3)
    assert 3 not in set(wl.seq_task.tolist())
    t = synth.layer_tensors(wl, 128, 128, seed=17)
    got = run_lib("bf16", wl, t, 128, 128)
    check_all(wl, oracle_inputs("bf16", t), got, BF16_TOL, 128, 128)


def test_bf16_c2_q_projection_full_size():
    """BASELINE config 2 at full size (T = 16384, 4 tasks r=16, s=2), the q projection
    4096 -> 4096 in the launch configuration bench.py times: dA_t/dB_t compared in
    full, Y/dX on sampled rows (every 64th row + all rows of the first sequence)."""
    wl = synth.config_c2()
    d_in = d_out = 4096
    t = synth.layer_tensors(wl, d_in, d_out, seed=21)
    Y, dX, dA, dB, _ = run_lib("bf16", wl, t, d_in, d_out)
    ti = oracle_inputs("bf16", t)
    rows = np.unique(np.concatenate([np.arange(0, wl.T, 64), np.arange(0, wl.seq_lens[0])]))
    # oracle on the sampled rows only (rows are independent)
    row_task = np.repeat(wl.seq_task, wl.seq_lens)[rows]
    lens1 = np.ones(len(rows), np.int32)
    args = (ti["X"][rows], ti["W"], ti["A"], ti["B"], wl.ranks.tolist(), wl.scales, lens1, row_task)
    Yo = O.lora_fwd(*args)
    dXo = O.lora_bwd(*args, ti["dY"][rows])[0]
    assert O.max_rel_err(Y[rows], Yo) < BF16_TOL
    assert O.max_rel_err(dX[rows], dXo) < BF16_TOL
    # full adapter gradients
    fargs = (ti["X"], ti["W"], ti["A"], ti["B"], wl.ranks.tolist(), wl.scales, wl.seq_lens, wl.seq_task)
    _, dAo, dBo = _bwd_adapters_only(*fargs, ti["dY"])
    roff = np.concatenate([[0], np.cumsum(wl.ranks)])
    for k in range(len(wl.ranks)):
        assert O.max_rel_err(dA[roff[k]:roff[k + 1]], dAo[roff[k]:roff[k + 1]]) < BF16_TOL
        assert O.max_rel_err(dB[:, roff[k]:roff[k + 1]], dBo[:, roff[k]:roff[k + 1]]) < BF16_TOL


def _bwd_adapters_only(X, W, A, B, ranks, scales, lens, tasks, dY):
    return O.lora_bwd(X, W, A, B, ranks, scales, lens, tasks, dY, want_dx=False)


def _full_size_check(wl, d_in, d_out, seed, row_stride):
    """Y/dX on sampled rows (every `row_stride`-th row + the first sequence), dA_t/dB_t
    in full, at the bench launch configuration."""
    t = synth.layer_tensors(wl, d_in, d_out, seed=seed)
    Y, dX, dA, dB, _ = run_lib("bf16", wl, t, d_in, d_out)
    ti = oracle_inputs("bf16", t)
    rows = np.unique(np.concatenate([np.arange(0, wl.T, row_stride), np.arange(0, wl.seq_lens[0])]))
    row_task = np.repeat(wl.seq_task, wl.seq_lens)[rows]
    args = (ti["X"][rows], ti["W"], ti["A"], ti["B"], wl.ranks.tolist(), wl.scales,
            np.ones(len(rows), np.int32), row_task)
    errs = {"Y": O.max_rel_err(Y[rows], O.lora_fwd(*args)),
            "dX": O.max_rel_err(dX[rows], O.lora_bwd(*args, ti["dY"][rows])[0])}
    fargs = (ti["X"], ti["W"], ti["A"], ti["B"], wl.ranks.tolist(), wl.scales, wl.seq_lens, wl.seq_task)
    _, dAo, dBo = _bwd_adapters_only(*fargs, ti["dY"])
    roff = np.concatenate([[0], np.cumsum(wl.ranks)])
    for k in range(len(wl.ranks)):
        if (wl.seq_task == k).any():
            errs[f"dA{k}"] = O.max_rel_err(dA[roff[k]:roff[k + 1]], dAo[roff[k]:roff[k + 1]])
            errs[f"dB{k}"] = O.max_rel_err(dB[:, roff[k]:roff[k + 1]], dBo[:, roff[k]:roff[k + 1]])
    bad = {k: v for k, v in errs.items() if not v < BF16_TOL}
    assert not bad, (bad, errs)


def test_bf16_c2_down_projection_full_size():
    """BASELINE config 2, the down projection 11008 -> 4096 (K = 172 blocks of 64)."""
    _full_size_check(synth.config_c2(), 11008, 4096, seed=22, row_stride=97)


def test_bf16_c3_q_projection_full_size():
    """BASELINE config 3: 16 tasks, ranks 8/16/32/64, scales 0.5/1/2/4, long-tail lengths
    up to 16K packed into T = 65536, q projection 4096 -> 4096."""
    _full_size_check(synth.config_c3(), 4096, 4096, seed=23, row_stride=211)


def _wl(lens, tasks, ranks, scales):
    ts = [synth.TaskSpec(f"t{i}", 0, 0, 1, r, s) for i, (r, s) in enumerate(zip(ranks, scales))]
    return synth.Workload("edge", ts, np.array(lens, np.int32), np.array(tasks, np.int32), 0)


@pytest.mark.parametrize("case", [
    # (lens, tasks, ranks, scales, in, out)
    ([1], [0], [16], [2.0], 64, 64),                                   # one token
    ([0, 5, 0, 3], [1, 0, 1, 0], [8, 4], [1.0, 3.0], 128, 64),         # zero-length seqs, task w/o tokens
    ([3, 2, 4, 1, 5, 2, 3, 1, 2, 6], list(range(10)), [1, 2, 3, 5, 7, 9, 11, 13, 17, 64],
     [0.5, 1, 2, 4, 0.5, 1, 2, 4, 0.5, 1], 192, 320),                  # 10 tasks in one tile, odd ranks (B padding path)
    ([130, 1, 127, 256, 2], [2, 0, 1, 2, 0], [64, 64, 64], [1.0, 1.0, 1.0], 64, 128),  # rank 64, one K block
    ([300] * 3 + [7] * 20, [0, 1, 2] + [i % 3 for i in range(20)], [16, 32, 48], [2.0, 1.0, 0.5], 256, 256),
    # 64 tasks, 2-9 tokens each, interleaved (up to ~30 task slots per 128-row tile, every
    # pair tile's union of tasks in the K-extension), ranks cycling 4..64
    ([2 + (i * 7) % 8 for i in range(64)], [(i * 37) % 64 for i in range(64)],
     [4 * (1 + i % 16) for i in range(64)], [0.5 + 0.25 * (i % 4) for i in range(64)], 128, 192),
])
def test_bf16_edge_cases(case):
    lens, tasks, ranks, scales, d_in, d_out = case
    wl = _wl(lens, tasks, ranks, scales)
    t = synth.layer_tensors(wl, d_in, d_out, seed=31)
    check_all(wl, oracle_inputs("bf16", t), run_lib("bf16", wl, t, d_in, d_out), BF16_TOL, d_in, d_out)


@pytest.mark.parametrize("case", [
    ([1], [0], [16], [2.0], 7, 5),
    ([0, 5, 0, 3, 40], [1, 0, 1, 0, 2], [8, 4, 1], [1.0, 3.0, -2.0], 33, 70),
])
def test_fp32_edge_cases(case):
    lens, tasks, ranks, scales, d_in, d_out = case
    wl = _wl(lens, tasks, ranks, scales)
    t = synth.layer_tensors(wl, d_in, d_out, seed=32)
    check_all(wl, oracle_inputs("fp32", t), run_lib("fp32", wl, t, d_in, d_out), FP32_TOL, d_in, d_out)


def test_bf16_deterministic():
    """Two identical calls give bit-identical outputs (fixed-order reductions, no atomics
    in the value path)."""
    wl = _medium(seed=12)
    t = synth.layer_tensors(wl, 256, 256, seed=33)
    a = run_lib("bf16", wl, t, 256, 256)
    b = run_lib("bf16", wl, t, 256, 256)
    for x, y in zip(a[:4], b[:4]):
        assert np.array_equal(x, y)


def test_abi_rejects_bad_input_before_launch():
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    dev = torch.device("cuda:0")
    X = torch.zeros(4, 100, device=dev, dtype=torch.bfloat16)     # in not a multiple of 64
    W = torch.zeros(64, 100, device=dev, dtype=torch.bfloat16)
    with pytest.raises(_lib.LobraError) as e:
        _lib.lobra_lora_fwd(X, W, W, W, [4], [1.0], [4], [0], X, X, X, ws_bytes=1 << 20)
    assert e.value.status == _lib.LOBRA_ERR_INPUT
    X = torch.zeros(4, 64, device=dev, dtype=torch.bfloat16)
    W = torch.zeros(64, 64, device=dev, dtype=torch.bfloat16)
    with pytest.raises(_lib.LobraError) as e:                        # task id out of range
        _lib.lobra_lora_fwd(X, W, W, W, [4], [1.0], [4], [3], X, X, X, ws_bytes=1 << 20)
    assert e.value.status == _lib.LOBRA_ERR_INPUT
    with pytest.raises(_lib.LobraError) as e:                        # rank 65
        _lib.lobra_lora_fwd(X, W, W, W, [65], [1.0], [4], [0], X, X, X, ws_bytes=1 << 20)
    assert e.value.status == _lib.LOBRA_ERR_INPUT


def test_empty_batch():
    """T = 0 (every sequence empty): forward is a no-op, backward writes zero adapter
    gradients (reading Q10) and leaves dX alone."""
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    dev = torch.device("cuda:0")
    for code, td in ((_lib.LOBRA_BF16, torch.bfloat16), (_lib.LOBRA_FP32, torch.float32)):
        X = torch.zeros(1, 64, device=dev, dtype=td)
        W = torch.zeros(64, 64, device=dev, dtype=td)
        A = torch.zeros(8, 64, device=dev, dtype=td)
        B = torch.zeros(64, 8, device=dev, dtype=td)
        ws = torch.empty(_lib.lobra_lora_workspace_bytes(code, 64, 64, [0, 0], [0, 1], [4, 4], [1, 1]),
                         dtype=torch.uint8, device=dev)
        Hs = torch.empty(_lib.lobra_lora_saved_bytes(code, 64, 64, [0, 0], [0, 1], [4, 4], [1, 1]),
                         dtype=torch.uint8, device=dev)
        _lib.lobra_lora_fwd(X, W, A, B, [4, 4], [1, 1], [0, 0], [0, 1], X, Hs, ws)
        dA = torch.full((8, 64), 7.0, device=dev)
        dB = torch.full((64, 8), 7.0, device=dev)
        _lib.lobra_lora_bwd(X, W, A, B, [4, 4], [1, 1], [0, 0], [0, 1], Hs, X, X, dA, dB, ws)
        torch.cuda.synchronize()
        assert not dA.any() and not dB.any()
        dA.fill_(7.0)
        _lib.lobra_lora_bwd(X, W, A, B, [4, 4], [1, 1], [0, 0], [0, 1], Hs, X, X, dA, dB, ws,
                            accumulate_dadb=True)
        torch.cuda.synchronize()
        assert (dA == 7.0).all()


def test_workspace_too_small_is_rejected():
    torch = _torch()
    from paper_2509_01193_b200 import _lib
    dev = torch.device("cuda:0")
    X = torch.zeros(300, 128, device=dev, dtype=torch.bfloat16)
    W = torch.zeros(128, 128, device=dev, dtype=torch.bfloat16)
    A = torch.zeros(16, 128, device=dev, dtype=torch.bfloat16)
    B = torch.zeros(128, 16, device=dev, dtype=torch.bfloat16)
    ws = torch.empty(1024, dtype=torch.uint8, device=dev)
    with pytest.raises(_lib.LobraError) as e:
        _lib.lobra_lora_fwd(X, W, A, B, [16], [1.0], [300], [0], X, X, ws)
    assert e.value.status == _lib.LOBRA_ERR_INPUT and "workspace" in str(e.value)


@pytest.mark.parametrize("T,mixed", [
    (14080, False),   # 110 tiles: below 3/4 of the SMs -> split-K k_rowproj
    (14208, False),   # 111 tiles: k_shrink, one CTA per slot (slots fit one wave)
    (14300, False),   # 112 tiles, ragged last tile (92 rows)
    (16384, True),    # 128 tiles, 24 interleaved tasks: slots >> SMs -> k_shrink per tile,
                      # several passes of <= 4 slots per tile, many dY-pass segments
])
def test_bf16_shrink_paths_full_batch(T, mixed):
    """The forward-shrink variants and the balanced dY-pass schedule at bench-sized batches
    (every row, every task checked against the oracle; narrow widths keep it fast)."""
    rng = np.random.default_rng(T)
    if mixed:
        G = 24
        ranks = [8, 16, 32, 64] * 6
        lens = []
        while sum(lens) < T:
            lens.append(int(rng.integers(5, 90)))
        lens[-1] -= sum(lens) - T
        tasks = [(i * 7) % G for i in range(len(lens))]   # interleaved: many tasks per tile
    else:
        G = 4
        ranks = [16] * 4
        lens = [T // 8] * 8
        lens[-1] += T - sum(lens)
        tasks = [0, 0, 1, 1, 2, 2, 3, 3]
    scales = [0.5 + 0.5 * (i % 4) for i in range(G)]
    wl = _wl(lens, tasks, ranks, scales)
    assert wl.T == T
    t = synth.layer_tensors(wl, 256, 192, seed=41)
    check_all(wl, oracle_inputs("bf16", t), run_lib("bf16", wl, t, 256, 192), BF16_TOL, 256, 192)
