"""GPU parity of what bench.py times: LoraLayer's seven-projection step against the oracle.

bench.py runs `LoraLayer.forward` / `.backward` (projection-group calls for q/k/v and
gate/up, single calls for o and down, several chunks per step with accumulate_dadb, every
projection's dA/dB written at its offsets of the flat gradient buffer).  Here that exact
code path runs at full size and is compared with oracle/lora.py (fp64, the plain
definition of P:231 / the backward of SURVEY §8(c) c1):
  * Y and dX on sampled sequences (first, last, longest, three random ones; the oracle's
    rows are independent per sequence, so a sub-batch of whole sequences is exact);
  * every projection's per-task dA_t / dB_t read back from flat_grad, summed over BOTH
    chunks (accumulate_dadb), against the oracle's sum over all sequences of both chunks
    (computed sub-batch by sub-batch: the gradients are sums over sequences, reading Q7);
at the north-star tolerance 2e-2 (max |g - o| / max |o| per tensor, per task: reading Q9).
"""
import numpy as np
import pytest

from oracle import lora as O
from workloads import synth

pytestmark = pytest.mark.gpu

TOL = 2e-2


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _f64(t):
    return t.float().cpu().numpy().astype(np.float64)


def _sample_seqs(wl, rng, k=3):
    n = len(wl.seq_lens)
    pick = {0, n - 1, int(np.argmax(wl.seq_lens))}
    pick |= set(int(x) for x in rng.choice(n, size=min(k, n), replace=False))
    return sorted(pick)


def _rows_of(wl, seqs, edge=256):
    """Rows of the sampled sequences: all of a short one, the first and last `edge` rows of
    a long one (rows are independent, so each piece is its own 'sequence' for the oracle).
    Returns (rows, sub-batch lengths, sub-batch tasks)."""
    off = np.concatenate([[0], np.cumsum(wl.seq_lens)])
    rows, lens, tasks = [], [], []
    for s in seqs:
        a, b = int(off[s]), int(off[s + 1])
        parts = [(a, b)] if b - a <= 2 * edge else [(a, a + edge), (b - edge, b)]
        for x, y in parts:
            rows.append(np.arange(x, y))
            lens.append(y - x)
            tasks.append(int(wl.seq_task[s]))
    return np.concatenate(rows), np.array(lens, np.int32), np.array(tasks, np.int32)


def _run(shapes, ranks, scales, chunks, seed):
    """Runs the layer over the chunks (fresh io per chunk, dA/dB accumulated over chunks);
    returns per chunk (io host copies of sampled rows, Y rows, dX rows) and the flat grad."""
    torch = _torch()
    from paper_2509_01193_b200.layer import LoraLayer
    dev = torch.device("cuda:0")
    layer = LoraLayer(shapes, ranks, scales, dev, torch.bfloat16, seed=seed)
    rng = np.random.default_rng(seed)
    out = []
    for ci, wl in enumerate(chunks):
        T = wl.T
        io = layer.alloc_io(T, seed=seed * 10 + ci)
        lens, tsk = wl.seq_lens.astype(np.int32), wl.seq_task.astype(np.int32)
        layer.forward(lens, tsk, io, T)
        torch.cuda.synchronize()
        seqs = _sample_seqs(wl, rng)
        rows_np, sub_l, sub_t = _rows_of(wl, seqs)
        rows = torch.as_tensor(rows_np, device=dev)
        Y = {p.name: _f64(io["Y"][p.name][rows]) for p in layer.projs}
        layer.backward(lens, tsk, io, T, accumulate_dadb=ci > 0)
        torch.cuda.synchronize()
        dX = {g: _f64(io["dX"][g][rows]) for g in layer.groups()}
        out.append({"wl": wl, "io": io, "sub": (sub_l, sub_t), "rows": rows, "Y": Y, "dX": dX})
    return layer, out


def _check(layer, runs, ranks, scales, sub_rows=4096):
    torch = _torch()
    roff = np.concatenate([[0], np.cumsum(ranks)])
    fg = layer.flat_grad
    for p in layer.projs:
        W, A, B = _f64(p.W), _f64(p.A), _f64(p.B)
        dA_ref = np.zeros_like(A)
        dB_ref = np.zeros_like(B)
        for run in runs:
            wl, io = run["wl"], run["io"]
            X_all, dY_all = io["X"][p.group], io["dY"][p.name]
            # sampled sequences: Y rows
            sub_l, sub_t = run["sub"]
            x = _f64(X_all[run["rows"]])
            Yo = O.lora_fwd(x, W, A, B, ranks, scales, sub_l, sub_t)
            e = O.max_rel_err(run["Y"][p.name], Yo)
            assert e <= TOL, (p.name, "Y", e)
            # all sequences, sub-batch by sub-batch: dA / dB sums
            off = np.concatenate([[0], np.cumsum(wl.seq_lens)])
            s0 = 0
            while s0 < len(wl.seq_lens):
                s1 = s0
                while s1 < len(wl.seq_lens) and off[s1 + 1] - off[s0] <= max(sub_rows, wl.seq_lens[s0]):
                    s1 += 1
                a, b = int(off[s0]), int(off[s1])
                _, dA_s, dB_s = O.lora_bwd(_f64(X_all[a:b]), W, A, B, ranks, scales, wl.seq_lens[s0:s1],
                                           wl.seq_task[s0:s1], _f64(dY_all[a:b]), want_dx=False)
                dA_ref += dA_s
                dB_ref += dB_s
                s0 = s1
        R = int(roff[-1])
        dA = fg[p.dA_off:p.dA_off + R * p.d_in].view(R, p.d_in).double().cpu().numpy()
        dB = fg[p.dB_off:p.dB_off + p.d_out * R].view(p.d_out, R).double().cpu().numpy()
        for t in range(len(ranks)):
            r0, r1 = int(roff[t]), int(roff[t + 1])
            if not np.any(dA_ref[r0:r1]):
                assert not np.any(dA[r0:r1]) and not np.any(dB[:, r0:r1]), (p.name, t, "task without tokens")
                continue
            ea = O.max_rel_err(dA[r0:r1], dA_ref[r0:r1])
            eb = O.max_rel_err(dB[:, r0:r1], dB_ref[:, r0:r1])
            assert ea <= TOL and eb <= TOL, (p.name, t, ea, eb)
    # dX of every input group = sum over its projections (sampled sequences, each chunk)
    for run in runs:
        io = run["io"]
        sub_l, sub_t = run["sub"]
        for g in layer.groups():
            ref = None
            for p in layer.members(g):
                W, A, B = _f64(p.W), _f64(p.A), _f64(p.B)
                dXo, _, _ = O.lora_bwd(_f64(io["X"][g][run["rows"]]), W, A, B, ranks, scales, sub_l, sub_t,
                                       _f64(io["dY"][p.name][run["rows"]]))
                ref = dXo if ref is None else ref + dXo
            e = O.max_rel_err(run["dX"][g], ref)
            assert e <= TOL, (g, "dX", e)


def test_c2_layer_two_chunks_vs_oracle():
    """C2 (BASELINE configs[1]): all seven Llama-2-7B projections (gate/up 4096 -> 11008,
    down 11008 -> 4096), a full T = 16384 chunk then a second 8192-token chunk
    accumulating dA/dB, exactly as bench.py drives the layer."""
    from paper_2509_01193_b200.layer import LLAMA2_7B
    tasks = synth.c2_tasks()
    ranks, scales = [t.rank for t in tasks], [t.scale for t in tasks]
    chunks = [synth.config_c2(seed=2), synth.config_c2(seed=5, t_max=8192)]
    layer, runs = _run(LLAMA2_7B, ranks, scales, chunks, seed=21)
    _check(layer, runs, ranks, scales)


def test_c3_qkv_gate_up_vs_oracle():
    """C3 (BASELINE configs[2]): 16 tasks with ranks 8..64 (wide projection groups: the
    planes shrink), T = 65536 with sequences up to 16K, q/k/v and gate/up through the
    group calls."""
    from paper_2509_01193_b200.layer import LLAMA2_7B
    tasks = synth.c3_tasks()
    ranks, scales = [t.rank for t in tasks], [t.scale for t in tasks]
    shapes = [s for s in LLAMA2_7B if s[0] in ("q", "k", "v", "gate", "up")]
    layer, runs = _run(shapes, ranks, scales, [synth.config_c3(seed=3)], seed=33)
    _check(layer, runs, ranks, scales, sub_rows=8192)


def test_c3_o_down_vs_oracle():
    """C3 (BASELINE configs[2]): the single-call projections, o (4096 -> 4096) and down
    (11008 -> 4096, the K = 11008 GEMMs and the widest X of the dA reduction), 16 tasks with
    ranks 8..64, T = 65536 with sequences up to 16K -- with the group test above, every
    projection bench.py times on C3 is compared with the oracle at full size."""
    from paper_2509_01193_b200.layer import LLAMA2_7B
    tasks = synth.c3_tasks()
    ranks, scales = [t.rank for t in tasks], [t.scale for t in tasks]
    shapes = [s for s in LLAMA2_7B if s[0] in ("o", "down")]
    layer, runs = _run(shapes, ranks, scales, [synth.config_c3(seed=4)], seed=34)
    _check(layer, runs, ranks, scales, sub_rows=8192)


def test_launch_counter_matches_cupti():
    """lobra_launch_count (the bench's `gpu_launches`) counts every kernel the library
    enqueues -- the dY pass's G finalize included -- as CUPTI sees them."""
    torch = _torch()
    from torch.profiler import ProfilerActivity, profile
    from paper_2509_01193_b200 import _lib
    from paper_2509_01193_b200.layer import LLAMA2_7B, LoraLayer
    tasks = synth.c2_tasks()
    ranks, scales = [t.rank for t in tasks], [t.scale for t in tasks]
    shapes = [(n, i // 4, o // 4, k, g) for n, i, o, k, g in LLAMA2_7B]
    layer = LoraLayer(shapes, ranks, scales, torch.device("cuda:0"), torch.bfloat16, seed=3)
    wl = synth.config_c2(seed=9, t_max=4096)
    io = layer.alloc_io(wl.T, seed=4)
    lens, tsk = wl.seq_lens.astype(np.int32), wl.seq_task.astype(np.int32)
    layer.forward(lens, tsk, io, wl.T)            # warm (workspace allocation, attributes)
    layer.backward(lens, tsk, io, wl.T, accumulate_dadb=False)
    torch.cuda.synchronize()
    n0 = _lib.lobra_launch_count()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        layer.forward(lens, tsk, io, wl.T)
        layer.backward(lens, tsk, io, wl.T, accumulate_dadb=False)
        torch.cuda.synchronize()
    n = _lib.lobra_launch_count() - n0
    kern = [e for e in prof.events() if e.device_type.name == "CUDA" and not e.name.startswith(("Memcpy", "Memset"))]
    assert n == len(kern) > 0, (n, sorted({e.name.split("(")[0] for e in kern}))
