"""GPU: pipeline-parallel execution (paper_2509_01193_b200/pipeline.py; SURVEY NEXT-3, App. D
P:1499-1532).  Two stages (one decoder layer each, two processes, gloo with host staging,
both on cuda:0 -- a correctness test of the 1F1B executor, not a timing) run four
variable-length packed micro-batches; the last stage's outputs, the first stage's input
gradients and both layers' adapter gradients equal, bit for bit, a single-process run of
the same two layers (every forward, then every backward in micro-batch order)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SMALL = [("q", 256, 256, "col", "attn"), ("k", 256, 256, "col", "attn"), ("v", 256, 256, "col", "attn"),
         ("o", 256, 256, "row", "o_in"), ("gate", 256, 512, "col", "mlp"), ("up", 256, 512, "col", "mlp"),
         ("down", 512, 256, "row", "down_in")]
MICRO = [([300, 57, 1], [0, 1, 1]), ([129, 200], [1, 0]), ([33, 77, 12], [0, 0, 1]), ([256], [1])]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layer(seed):
    from paper_2509_01193_b200.decoder import DecoderLayer
    layer = DecoderLayer(SMALL, n_heads=2, ranks=[16, 8], scales=[2.0, 0.5], seed=seed,
                         deterministic_attn=True, attn_backend="flash_attn")
    for p in layer.lora.projs:
        p.B.mul_(0.25)
    return layer


def _data():
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(42)
    xs, gs = [], []
    for lens, _ in MICRO:
        T = sum(lens)
        xs.append(torch.randn(T, 256, generator=g, device="cuda").to(torch.bfloat16))
        gs.append(torch.randn(T, 256, generator=g, device="cuda").to(torch.bfloat16))
    return xs, gs


def _np(t):
    return t.float().cpu().numpy()


def _worker(rank, port, q):
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=2)
        torch.cuda.set_device(0)
        from paper_2509_01193_b200.pipeline import PipelineStage
        micro = [(np.array(l, np.int32), np.array(t, np.int32)) for l, t in MICRO]
        xs, gs = _data()
        layer = _layer(100 + rank)
        st = PipelineStage([layer], rank, 2, prev=0 if rank == 1 else None, next=1 if rank == 0 else None,
                           host_staging=True)
        outs, dxs = st.run(micro, inputs=xs if rank == 0 else None, grads=gs if rank == 1 else None)
        torch.cuda.synchronize()
        res = {"flat": _np(layer.lora.flat_grad)}
        if rank == 1:
            res["Y"] = [_np(outs[k]) for k in range(len(micro))]
        else:
            res["dX"] = [_np(dxs[k]) for k in range(len(micro))]
            # single-process reference: the same two layers, all forwards then all backwards
            l0, l1 = _layer(100), _layer(101)
            ys = []
            for k, (lens, tasks) in enumerate(micro):
                for lay in (l0, l1):
                    lay.select_context(k)
                ys.append(l1.forward(lens, tasks, l0.forward(lens, tasks, xs[k])))
            ref_dx = []
            for k, (lens, tasks) in enumerate(micro):
                for lay in (l0, l1):
                    lay.select_context(k)
                ref_dx.append(l0.backward(l1.backward(gs[k], accumulate_dadb=k > 0), accumulate_dadb=k > 0))
            torch.cuda.synchronize()
            res["ref"] = {"Y": [_np(y) for y in ys], "dX": [_np(d) for d in ref_dx],
                          "flat0": _np(l0.lora.flat_grad), "flat1": _np(l1.lora.flat_grad)}
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_two_stage_1f1b_equals_single_process():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    pytest.importorskip("flash_attn")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r in (0, 1):
        assert isinstance(res[r], dict), res[r]
    ref = res[0]["ref"]
    for k in range(len(MICRO)):
        assert np.array_equal(res[1]["Y"][k], ref["Y"][k]), k
        assert np.array_equal(res[0]["dX"][k], ref["dX"][k]), k
    assert np.array_equal(res[0]["flat"], ref["flat0"])
    assert np.array_equal(res[1]["flat"], ref["flat1"])
