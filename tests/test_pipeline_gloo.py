"""Pipeline-parallel executor (`pipeline.PipelineStage`, 1F1B over variable-length
micro-batches; App. D) on CPU with gloo: 3 stages on 3 processes.

The stages hold stand-in layers (a per-layer affine map on bf16 rows, with a saved input
per micro-batch and a gradient that the first micro-batch overwrites and later ones
accumulate), so what is under test is the executor's own logic: the 1F1B op order per
stage, the point-to-point shapes for micro-batches of different lengths, the per-micro-batch
context switch, and the gradient accumulation order.  Every output, input gradient and layer
gradient must equal a single-process run of the same layers bit for bit.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

H = 24
MICRO = [([5, 9], [0, 1]), ([17], [1]), ([3, 4, 2], [0, 0, 1]), ([11, 1], [1, 0]), ([6], [0])]


class AffineLayer:
    """y = x * w + b (bf16); backward: dx = g * w, grad (+)= sum over rows of g * x."""

    def __init__(self, idx):
        self.h, self.dev = H, torch.device("cpu")
        gen = torch.Generator().manual_seed(100 + idx)
        self.w = (torch.rand(H, generator=gen) + 0.5).to(torch.bfloat16)
        self.b = (torch.rand(H, generator=gen) - 0.5).to(torch.bfloat16)
        self.saved, self.k = {}, None
        self.grad = torch.zeros(H, dtype=torch.float32)
        self.log = []

    def select_context(self, k):
        self.k = k

    def forward(self, lens, tasks, x):
        assert x.shape == (sum(lens), H) and x.dtype == torch.bfloat16
        self.saved[self.k] = x
        self.log.append(("F", self.k))
        return x * self.w + self.b

    def backward(self, g, accumulate_dadb=False):
        x = self.saved.pop(self.k)
        assert g.shape == x.shape
        self.log.append(("B", self.k))
        part = (g.float() * x.float()).sum(0)
        self.grad = self.grad + part if accumulate_dadb else part
        return g * self.w


def _inputs():
    gen = torch.Generator().manual_seed(7)
    xs = [torch.randn(sum(l), H, generator=gen).to(torch.bfloat16) for l, _ in MICRO]
    gs = [torch.randn(sum(l), H, generator=gen).to(torch.bfloat16) for l, _ in MICRO]
    return xs, gs


def _stage_layers(stage, per_stage=2):
    return [AffineLayer(stage * per_stage + i) for i in range(per_stage)]


def _reference(num_stages):
    """All layers in one process: forward of every micro-batch, then backwards in order."""
    layers = [l for s in range(num_stages) for l in _stage_layers(s)]
    xs, gs = _inputs()
    outs, dxs = {}, {}
    for k, (lens, tasks) in enumerate(MICRO):
        x = xs[k]
        for l in layers:
            l.select_context(k)
            x = l.forward(lens, tasks, x)
        outs[k] = x
    for k in range(len(MICRO)):
        g = gs[k]
        for l in reversed(layers):
            l.select_context(k)
            g = l.backward(g, accumulate_dadb=k > 0)
        dxs[k] = g
    return outs, dxs, [l.grad for l in layers]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, host_staging, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2509_01193_b200.pipeline import PipelineStage, schedule_1f1b

        layers = _stage_layers(rank)
        st = PipelineStage(layers, rank, world, prev=rank - 1 if rank > 0 else None,
                           next=rank + 1 if rank < world - 1 else None, host_staging=host_staging)
        xs, gs = _inputs()
        outs, dxs = st.run(MICRO, inputs=xs if rank == 0 else None, grads=gs if rank == world - 1 else None)
        # every layer of the stage saw the stage's 1F1B order, and no activation is left over
        order = schedule_1f1b(world, rank, len(MICRO))
        assert all(l.log == order for l in layers), (layers[0].log, order)
        assert all(not l.saved for l in layers)
        # plain arrays through the queue (bf16 -> fp32 is exact): torch tensors would travel
        # as shared-memory handles that die with this process
        npy = lambda d: {k: v.float().numpy() for k, v in d.items()}
        q.put((rank, {"outs": npy(outs), "dxs": npy(dxs), "grads": [l.grad.numpy() for l in layers]}))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("host_staging", [False, True])
def test_pipeline_1f1b_gloo_world3(host_staging):
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, host_staging, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert isinstance(res[r], dict), res[r]
    ref_outs, ref_dxs, ref_grads = _reference(world)
    last, first = res[world - 1], res[0]
    assert sorted(last["outs"]) == list(range(len(MICRO))) and not res[1]["outs"]
    assert sorted(first["dxs"]) == list(range(len(MICRO))) and not res[1]["dxs"]
    for k in range(len(MICRO)):
        assert torch.equal(torch.from_numpy(last["outs"][k]), ref_outs[k].float())
        assert torch.equal(torch.from_numpy(first["dxs"][k]), ref_dxs[k].float())
    got = [g for r in range(world) for g in res[r]["grads"]]
    assert len(got) == len(ref_grads)
    for a, b in zip(got, ref_grads):
        assert torch.equal(torch.from_numpy(a), b)
