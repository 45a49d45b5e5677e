"""N > 1 host logic on CPU with torch.distributed gloo, world_size 2.

* every rank computes the identical dispatch locally (no broadcast needed);
* data-parallel replicas: per-rank gradients of their dispatched sequences, written into
  the full-size flat buffer and SUM-all-reduced, equal the full-batch gradients;
* tensor-parallel replica (TP2): the column/row shards and the gradient offsets used by
  ``layer.LoraLayer`` give, after the collectives the library issues (row: Y all-reduce;
  column: dX all-reduce) and the adapter all-reduce, exactly the unsharded result -- LoRA
  adds no collective of its own.
The per-shard arithmetic is the fp64 oracle (test infrastructure); what is under test is
the decomposition, offsets and reduction plumbing the GPU path uses.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tiny(seed):
    rng = np.random.default_rng(seed)
    d_in, d_out, ranks, scales = 16, 12, [3, 5], [2.0, 0.5]
    lens = np.array([5, 9, 3, 7, 6, 4], np.int32)
    tasks = np.array([0, 1, 1, 0, 1, 0], np.int32)
    T, R = int(lens.sum()), sum(ranks)
    return dict(X=rng.standard_normal((T, d_in)), W=rng.standard_normal((d_out, d_in)),
                A=rng.standard_normal((R, d_in)), B=rng.standard_normal((d_out, R)),
                dY=rng.standard_normal((T, d_out)), lens=lens, tasks=tasks, ranks=ranks,
                scales=scales, d_in=d_in, d_out=d_out)


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import lora as O
        from paper_2509_01193_b200 import _lib
        from paper_2509_01193_b200.layer import grad_offsets, shard
        from workloads import synth

        # 1. identical dispatch on every rank
        wl = synth.sample_batch(synth.c2_tasks(), seed=5, l_max=4096, per_task=[16, 8, 8, 4])
        d = _lib.lobra_dispatch([1, 2], [2, 1], [4096, 8192], [[k + 1 for k in range(32)],
                                [max(1, (k + 1) // 2) for k in range(32)]],
                                wl.seq_lens, wl.seq_task, 256, 8192, 8, 0, chunking=1)
        got = [None] * world
        dist.all_gather_object(got, {k: (v.tolist() if hasattr(v, "tolist") else v) for k, v in d.items()})
        assert all(g == got[0] for g in got), "ranks disagree on the dispatch"

        p = _tiny(7)
        X, W, A, B, dY = p["X"], p["W"], p["A"], p["B"], p["dY"]
        lens, tasks, ranks, scales = p["lens"], p["tasks"], p["ranks"], p["scales"]
        d_in, d_out, R = p["d_in"], p["d_out"], sum(ranks)
        full = O.lora_bwd(X, W, A, B, ranks, scales, lens, tasks, dY)
        Yfull = O.lora_fwd(X, W, A, B, ranks, scales, lens, tasks)

        # 2. data parallel: 2 x TP1, sequences split by rank (round robin)
        offs = np.concatenate([[0], np.cumsum(lens)])
        mine = [k for k in range(len(lens)) if k % world == rank]
        rows = np.concatenate([np.arange(offs[k], offs[k + 1]) for k in mine])
        _, dA, dB = O.lora_bwd(X[rows], W, A, B, ranks, scales, lens[mine], tasks[mine], dY[rows])
        flat = torch.tensor(np.concatenate([dA.ravel(), dB.ravel()]))
        dist.all_reduce(flat)
        fa, fb = flat[:R * d_in].numpy().reshape(R, d_in), flat[R * d_in:].numpy().reshape(d_out, R)
        assert np.allclose(fa, full[1], rtol=1e-12, atol=1e-12)
        assert np.allclose(fb, full[2], rtol=1e-12, atol=1e-12)

        # 3. one TP2 replica: column- and row-parallel shards
        for kind in ("col", "row"):
            si, so = shard(kind, world, rank, d_in, d_out)
            in_l, out_l = si.stop - si.start, so.stop - so.start
            Wl, Al, Bl = W[so, si], A[:, si], B[so]
            Xl = X[:, si]
            dYl = dY[:, so]
            Y = O.lora_fwd(Xl, Wl, Al, Bl, ranks, scales, lens, tasks)
            dXl, dAl, dBl = O.lora_bwd(Xl, Wl, Al, Bl, ranks, scales, lens, tasks, dYl)
            if kind == "row":      # library: forward Y all-reduce
                t = torch.tensor(Y)
                dist.all_reduce(t)
                assert np.allclose(t.numpy(), Yfull, atol=1e-10)
                parts = [None] * world
                dist.all_gather_object(parts, dXl)
                assert np.allclose(np.concatenate(parts, axis=1), full[0], atol=1e-10)
            else:                  # library: backward dX all-reduce
                parts = [None] * world
                dist.all_gather_object(parts, Y)
                assert np.allclose(np.concatenate(parts, axis=1), Yfull, atol=1e-10)
                t = torch.tensor(dXl)
                dist.all_reduce(t)
                assert np.allclose(t.numpy(), full[0], atol=1e-10)
            a_off, a_ld, b_off = grad_offsets(kind, rank, in_l, out_l, d_in, R)
            buf = np.zeros(R * d_in + d_out * R)
            dAv = buf[a_off:R * d_in]
            for r in range(R):
                dAv[r * a_ld:r * a_ld + in_l] += dAl[r]
            dBv = buf[R * d_in + b_off:]
            dBv[:out_l * R] += dBl.ravel()
            t = torch.tensor(buf)
            dist.all_reduce(t)                       # lobra_adapter_allreduce (SUM)
            ga = t[:R * d_in].numpy().reshape(R, d_in)
            gb = t[R * d_in:].numpy().reshape(d_out, R)
            assert np.allclose(ga, full[1], atol=1e-10), kind
            assert np.allclose(gb, full[2], atol=1e-10), kind
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
