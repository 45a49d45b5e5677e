"""NCCL plumbing on one GPU: a world-1 communicator with its TP sub-communicator
(ncclCommSplit), the TP all-reduces inside lobra_lora_fwd/bwd (COLUMN / ROW) and the
adapter-gradient all-reduce, with the collectives forced on 1-rank groups
(LOBRA_FORCE_COLLECTIVES=1).  A 1-rank SUM is the identity, so results must equal the
unsharded run bit for bit.  Run in a subprocess so the env var is set before the library
reads it."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
from paper_2509_01193_b200 import _lib
from workloads import synth
dev = torch.device("cuda:0")
torch.cuda.set_device(0)
uid = _lib.lobra_nccl_unique_id()
comm = _lib.lobra_comm_init(uid, 1, 0, 0)
assert (comm.tp_size, comm.tp_rank) == (1, 0)
lens, tasks, ranks, scales = [100, 60, 200], [0, 1, 0], [16, 8], [2.0, 0.5]
wl = synth.Workload("c", [synth.TaskSpec("a", 0, 0, 1, 16, 2.0), synth.TaskSpec("b", 0, 0, 1, 8, 0.5)],
                    np.array(lens, np.int32), np.array(tasks, np.int32), 0)
t = synth.layer_tensors(wl, 256, 192, seed=5)
d = {k: torch.from_numpy(synth.round_bf16(v)).to(dev).to(torch.bfloat16) for k, v in t.items()}
T = wl.T
code = _lib.LOBRA_BF16
ws = torch.empty(_lib.lobra_lora_workspace_bytes(code, 256, 192, lens, tasks, ranks, scales), dtype=torch.uint8, device=dev)
Hs = torch.empty(_lib.lobra_lora_saved_bytes(code, 256, 192, lens, tasks, ranks, scales), dtype=torch.uint8, device=dev)
outs = {}
for kind in (_lib.LOBRA_TP_NONE, _lib.LOBRA_TP_COLUMN, _lib.LOBRA_TP_ROW):
    c = None if kind == _lib.LOBRA_TP_NONE else comm
    Y = torch.empty(T, 192, dtype=torch.bfloat16, device=dev)
    dX = torch.empty(T, 256, dtype=torch.bfloat16, device=dev)
    dA = torch.empty(24, 256, dtype=torch.float32, device=dev)
    dB = torch.empty(192, 24, dtype=torch.float32, device=dev)
    _lib.lobra_lora_fwd(d["X"], d["W"], d["A"], d["B"], ranks, scales, lens, tasks, Y, Hs, ws, tp_kind=kind, comm=c)
    _lib.lobra_lora_bwd(d["X"], d["W"], d["A"], d["B"], ranks, scales, lens, tasks, Hs, d["dY"], dX, dA, dB, ws, tp_kind=kind, comm=c)
    flat = torch.cat([dA.flatten(), dB.flatten()]).contiguous()
    _lib.lobra_adapter_allreduce(comm, flat)
    torch.cuda.synchronize()
    outs[kind] = [x.float().cpu() for x in (Y, dX, dA, dB, flat)]
for kind in (_lib.LOBRA_TP_COLUMN, _lib.LOBRA_TP_ROW):
    for a, b in zip(outs[_lib.LOBRA_TP_NONE], outs[kind]):
        assert torch.equal(a, b), kind
# projection group (q/k/v-like, 3 bands) through the group calls: COLUMN all-reduces dX
# once, ROW every Y_p; with forced 1-rank collectives both equal the no-TP run
outs_g = [192, 128, 64]
tg = [synth.layer_tensors(wl, 256, o, seed=9 + p) for p, o in enumerate(outs_g)]
up = lambda a: torch.from_numpy(synth.round_bf16(a)).to(dev).to(torch.bfloat16)
Ws = [up(x["W"]) for x in tg]; As = [up(x["A"]) for x in tg]; Bs = [up(x["B"]) for x in tg]
dYs = [up(x["dY"]) for x in tg]
wsg = torch.empty(_lib.lobra_lora_group_workspace_bytes(code, 256, outs_g, lens, tasks, ranks, scales), dtype=torch.uint8, device=dev)
Hg = torch.empty(_lib.lobra_lora_group_saved_bytes(code, 256, outs_g, lens, tasks, ranks, scales), dtype=torch.uint8, device=dev)
res = {}
for kind in (_lib.LOBRA_TP_NONE, _lib.LOBRA_TP_COLUMN, _lib.LOBRA_TP_ROW):
    c = None if kind == _lib.LOBRA_TP_NONE else comm
    Ys = [torch.empty(T, o, dtype=torch.bfloat16, device=dev) for o in outs_g]
    dX = torch.empty(T, 256, dtype=torch.bfloat16, device=dev)
    dA = [torch.empty(24, 256, dtype=torch.float32, device=dev) for _ in outs_g]
    dB = [torch.empty(o, 24, dtype=torch.float32, device=dev) for o in outs_g]
    _lib.lobra_lora_group_fwd(d["X"], Ws, As, Bs, ranks, scales, lens, tasks, Ys, Hg, wsg, tp_kind=kind, comm=c)
    _lib.lobra_lora_group_bwd(d["X"], Ws, As, Bs, ranks, scales, lens, tasks, Hg, dYs, dX, dA, dB, wsg, tp_kind=kind, comm=c)
    torch.cuda.synchronize()
    res[kind] = [x.float().cpu() for x in Ys + [dX] + dA + dB]
for kind in (_lib.LOBRA_TP_COLUMN, _lib.LOBRA_TP_ROW):
    for a, b in zip(res[_lib.LOBRA_TP_NONE], res[kind]):
        assert torch.equal(a, b), ("group", kind)
comm.destroy()
print("COMM_OK")
'''


def test_world1_collectives_are_identity():
    pytest.importorskip("torch")
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, LOBRA_FORCE_COLLECTIVES="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT.replace("ROOT", repr(ROOT))], env=env,
                       capture_output=True, text=True, timeout=300)
    assert "COMM_OK" in r.stdout, r.stdout + r.stderr
