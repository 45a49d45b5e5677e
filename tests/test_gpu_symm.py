"""GPU: the own TP all-reduce over CUDA-IPC symmetric buffers, with two
processes on ONE GPU (peer buffers mapped through CUDA IPC exactly as across NVLink; the
handles travel over a gloo process group).  Checks:
  * bf16 / fp32 all-reduce over 3 epochs, ragged chunks: every rank's result is bitwise the
    rank-order fp32 sum of the partials, rounded once (computed on the host);
  * Megatron TP through the library's own collective (lobra_comm_from_symm, no NCCL): a
    row-parallel projection's forward Y (the FUSED GEMM -> reduce-scatter epilogue: output
    rows stored into their owner rank's buffer, bitwise equal to local GEMM + all-reduce,
    also for an odd T) and a column-parallel projection's / group's backward dX from 2
    shards equal the UNSHARDED fp64 oracle (bf16 tolerance) and are bitwise equal on both
    ranks.
"""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, ROOT)
from paper_2509_01193_b200 import _lib
from oracle import lora as O
from workloads import synth
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo", rank=rank, world_size=world)
dev = torch.device("cuda:0")
S = _lib.Symm(rank, world, 1 << 22)
hs = [None] * world
dist.all_gather_object(hs, S.handle)
S.open(hs)
# ---- raw all-reduce, bf16 and fp32, 3 epochs, ragged chunks
for it in range(3):
    for dt, n in ((torch.bfloat16, 8 * 12345), (torch.float32, 4 * 9999)):
        parts = [torch.randn(n, generator=torch.Generator().manual_seed(100 * it + r)).to(dt) for r in range(world)]
        x = parts[rank].to(dev)
        out = torch.empty_like(x)
        S.allreduce(x, out)
        torch.cuda.synchronize()
        acc = torch.zeros(n, dtype=torch.float32)
        for r in range(world):
            acc = acc + parts[r].float()
        ref = acc.to(dt)
        assert torch.equal(out.cpu(), ref), (it, dt, (out.cpu().float() - ref.float()).abs().max())
# ---- TP decomposition through lobra_comm_from_symm
comm = _lib.lobra_comm_from_symm(S)
lens, tasks, ranks, scales = [100, 60, 200], [0, 1, 0], [16, 8], [2.0, 0.5]
wl = synth.Workload("tp", [synth.TaskSpec("a", 0, 0, 1, 16, 2.0), synth.TaskSpec("b", 0, 0, 1, 8, 0.5)],
                    np.array(lens, np.int32), np.array(tasks, np.int32), 0)
d_in, d_out = 256, 256
t = synth.layer_tensors(wl, d_in, d_out, seed=5)
b = {k: synth.round_bf16(v) for k, v in t.items()}
o = {k: v.astype(np.float64) for k, v in b.items()}
up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(torch.bfloat16)
T = wl.T
args = (o["X"], o["W"], o["A"], o["B"], ranks, scales, lens, tasks)
Yo = O.lora_fwd(*args)
dXo, dAo, dBo = O.lora_bwd(*args, o["dY"])
code = _lib.LOBRA_BF16
# row-parallel (shard `in`): X, W columns, A columns
i0, i1 = rank * d_in // world, (rank + 1) * d_in // world
Xs, Ws, As = up(b["X"][:, i0:i1]), up(b["W"][:, i0:i1]), up(b["A"][:, i0:i1])
Bd = up(b["B"])
ws = torch.empty(_lib.lobra_lora_workspace_bytes(code, i1 - i0, d_out, lens, tasks, ranks, scales), dtype=torch.uint8, device=dev)
Hs = torch.empty(_lib.lobra_lora_saved_bytes(code, i1 - i0, d_out, lens, tasks, ranks, scales), dtype=torch.uint8, device=dev)
Y = torch.empty(T, d_out, dtype=torch.bfloat16, device=dev)
_lib.lobra_lora_fwd(Xs, Ws, As, Bd, ranks, scales, lens, tasks, Y, Hs, ws, tp_kind=_lib.LOBRA_TP_ROW, comm=comm)
torch.cuda.synchronize()
Yg = Y.float().cpu().numpy().astype(np.float64)
err = O.max_rel_err(Yg, Yo)
assert err <= 2e-2, ("row fwd", err)
# the fused GEMM -> reduce-scatter epilogue == local GEMM partial + own all-reduce, bitwise
Yp, Yr = torch.empty_like(Y), torch.empty_like(Y)
_lib.lobra_lora_fwd(Xs, Ws, As, Bd, ranks, scales, lens, tasks, Yp, Hs, ws)
S.allreduce(Yp, Yr)
torch.cuda.synchronize()
assert torch.equal(Yr, Y), "fused row-parallel forward differs from GEMM + all-reduce"
# odd T: unequal row chunks, 128-row tiles straddling the owner boundary
lens2 = [100, 61, 200]
wl2 = synth.Workload("tp2", wl.tasks, np.array(lens2, np.int32), np.array(tasks, np.int32), 0)
t2 = {k: synth.round_bf16(v) for k, v in synth.layer_tensors(wl2, d_in, d_out, seed=6).items()}
X2 = up(t2["X"][:, i0:i1])
ws2 = torch.empty(_lib.lobra_lora_workspace_bytes(code, i1 - i0, d_out, lens2, tasks, ranks, scales), dtype=torch.uint8, device=dev)
Hs2 = torch.empty(_lib.lobra_lora_saved_bytes(code, i1 - i0, d_out, lens2, tasks, ranks, scales), dtype=torch.uint8, device=dev)
Y2, Y2p, Y2r = (torch.empty(wl2.T, d_out, dtype=torch.bfloat16, device=dev) for _ in range(3))
W2, A2, B2 = up(t2["W"][:, i0:i1]), up(t2["A"][:, i0:i1]), up(t2["B"])
_lib.lobra_lora_fwd(X2, W2, A2, B2, ranks, scales, lens2, tasks, Y2, Hs2, ws2, tp_kind=_lib.LOBRA_TP_ROW, comm=comm)
_lib.lobra_lora_fwd(X2, W2, A2, B2, ranks, scales, lens2, tasks, Y2p, Hs2, ws2)
S.allreduce(Y2p, Y2r)
torch.cuda.synchronize()
assert torch.equal(Y2r, Y2)
o2 = {k: v.astype(np.float64) for k, v in t2.items()}
assert O.max_rel_err(Y2.float().cpu().numpy().astype(np.float64),
                     O.lora_fwd(o2["X"], o2["W"], o2["A"], o2["B"], ranks, scales, lens2, tasks)) <= 2e-2
# column-parallel (shard `out`): W rows, B rows; backward dX all-reduced
o0, o1 = rank * d_out // world, (rank + 1) * d_out // world
Wc, Bc, Ad = up(b["W"][o0:o1]), up(b["B"][o0:o1]), up(b["A"])
Xd, dYc = up(b["X"]), up(b["dY"][:, o0:o1])
ws = torch.empty(_lib.lobra_lora_workspace_bytes(code, d_in, o1 - o0, lens, tasks, ranks, scales), dtype=torch.uint8, device=dev)
Hs = torch.empty(_lib.lobra_lora_saved_bytes(code, d_in, o1 - o0, lens, tasks, ranks, scales), dtype=torch.uint8, device=dev)
Yc = torch.empty(T, o1 - o0, dtype=torch.bfloat16, device=dev)
dX = torch.empty(T, d_in, dtype=torch.bfloat16, device=dev)
dA = torch.empty(24, d_in, dtype=torch.float32, device=dev)
dB = torch.empty(o1 - o0, 24, dtype=torch.float32, device=dev)
_lib.lobra_lora_fwd(Xd, Wc, Ad, Bc, ranks, scales, lens, tasks, Yc, Hs, ws, tp_kind=_lib.LOBRA_TP_COLUMN, comm=comm)
_lib.lobra_lora_bwd(Xd, Wc, Ad, Bc, ranks, scales, lens, tasks, Hs, dYc, dX, dA, dB, ws, tp_kind=_lib.LOBRA_TP_COLUMN, comm=comm)
torch.cuda.synchronize()
dXg = dX.float().cpu().numpy().astype(np.float64)
err = O.max_rel_err(dXg, dXo)
assert err <= 2e-2, ("column bwd dX", err)
# fused GEMM -> reduce-scatter in the backward == local partial + own all-reduce, bitwise
dXp, dXr = torch.empty_like(dX), torch.empty_like(dX)
_lib.lobra_lora_bwd(Xd, Wc, Ad, Bc, ranks, scales, lens, tasks, Hs, dYc, dXp, dA, dB, ws)
S.allreduce(dXp, dXr)
torch.cuda.synchronize()
assert torch.equal(dXr, dX), "fused column-parallel backward differs from GEMM + all-reduce"
# both ranks hold bitwise the same all-reduced tensors
got = [None] * world
dist.all_gather_object(got, (Y.float().cpu().numpy().tobytes(), dX.float().cpu().numpy().tobytes()))
assert all(g == got[0] for g in got)
# the column-parallel adapter partials sum to the full gradients through the comm's world all-reduce
flat = torch.cat([dA.flatten(), torch.zeros(d_out * 24, device=dev)])
flat[24 * d_in + o0 * 24: 24 * d_in + o1 * 24] = dB.flatten()
_lib.lobra_adapter_allreduce(comm, flat)
torch.cuda.synchronize()
fa = flat[:24 * d_in].view(24, d_in).cpu().numpy().astype(np.float64)
fb = flat[24 * d_in:].view(d_out, 24).cpu().numpy().astype(np.float64)
assert O.max_rel_err(fa, dAo) <= 2e-2 and O.max_rel_err(fb, dBo) <= 2e-2
# projection group (q/k/v-like, column-parallel): the group's dX GEMMs accumulate in the
# symmetric stage area and one own all-reduce produces dX; row-parallel group forward
outs_full = [256, 128, 128]
tg = [synth.layer_tensors(wl, d_in, of, seed=9 + p) for p, of in enumerate(outs_full)]
bg = [{k: synth.round_bf16(v) for k, v in x.items()} for x in tg]
sh = [(rank * of // world, (rank + 1) * of // world) for of in outs_full]
Wg = [up(x["W"][a:c]) for x, (a, c) in zip(bg, sh)]
Ag = [up(x["A"]) for x in bg]
Bg = [up(x["B"][a:c]) for x, (a, c) in zip(bg, sh)]
dYg = [up(x["dY"][:, a:c]) for x, (a, c) in zip(bg, sh)]
outs_l = [c - a for a, c in sh]
wsg = torch.empty(_lib.lobra_lora_group_workspace_bytes(code, d_in, outs_l, lens, tasks, ranks, scales), dtype=torch.uint8, device=dev)
Hg = torch.empty(_lib.lobra_lora_group_saved_bytes(code, d_in, outs_l, lens, tasks, ranks, scales), dtype=torch.uint8, device=dev)
Ys = [torch.empty(T, ol, dtype=torch.bfloat16, device=dev) for ol in outs_l]
dXg = torch.empty(T, d_in, dtype=torch.bfloat16, device=dev)
dAs = [torch.empty(24, d_in, dtype=torch.float32, device=dev) for _ in outs_l]
dBs = [torch.empty(ol, 24, dtype=torch.float32, device=dev) for ol in outs_l]
Xg = up(bg[0]["X"])
_lib.lobra_lora_group_fwd(Xg, Wg, Ag, Bg, ranks, scales, lens, tasks, Ys, Hg, wsg, tp_kind=_lib.LOBRA_TP_COLUMN, comm=comm)
_lib.lobra_lora_group_bwd(Xg, Wg, Ag, Bg, ranks, scales, lens, tasks, Hg, dYg, dXg, dAs, dBs, wsg,
                          tp_kind=_lib.LOBRA_TP_COLUMN, comm=comm)
torch.cuda.synchronize()
ref = np.zeros((T, d_in))
og = [{k: v.astype(np.float64) for k, v in x.items()} for x in bg]
for x in og:
    ref += O.lora_bwd(og[0]["X"], x["W"], x["A"], x["B"], ranks, scales, lens, tasks, x["dY"])[0]
err = O.max_rel_err(dXg.float().cpu().numpy().astype(np.float64), ref)
assert err <= 2e-2, ("group column bwd dX", err)
got = [None] * world
dist.all_gather_object(got, dXg.float().cpu().numpy().tobytes())
assert all(g == got[0] for g in got)
# the group's last dX GEMM scatters (fused); == local group partial + own all-reduce, bitwise
dXgp, dXgr = torch.empty_like(dXg), torch.empty_like(dXg)
_lib.lobra_lora_group_bwd(Xg, Wg, Ag, Bg, ranks, scales, lens, tasks, Hg, dYg, dXgp, dAs, dBs, wsg)
S.allreduce(dXgp, dXgr)
torch.cuda.synchronize()
assert torch.equal(dXgr, dXg), "fused group backward differs from GEMM + all-reduce"
comm.destroy()
S.destroy()
print("SYMM_OK", rank)
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_symm_allreduce_and_tp_two_processes_one_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", SCRIPT.replace("ROOT", repr(ROOT))], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=300)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    for r, out in enumerate(outs):
        assert f"SYMM_OK {r}" in out, out[-3000:]
