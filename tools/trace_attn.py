"""Per-phase clock64 trace of CTA 0 of the attention backward (LOBRA_TRACE_ATTN=<file>):
one 4096-token sequence, so CTA 0 walks 32 query tiles.  Prints per-iteration phase
times in SM cycles relative to the iteration's S^T issue."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_01193_b200 import _lib  # noqa: E402

out = os.environ["LOBRA_TRACE_ATTN"]
lens = [4096]
T, H = sum(lens), 4
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, dO = (torch.randn(T, H, 128, generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
o = torch.empty_like(q)
lse = torch.empty(H, T, device="cuda")
ws = torch.empty(_lib.lobra_attn_workspace_bytes(lens, H), dtype=torch.uint8, device="cuda")
_lib.lobra_attn_fwd(np.array(lens, np.int32), q, k, v, o, lse, ws)
dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
wsb = torch.empty(_lib.lobra_attn_bwd_workspace_bytes(lens, H, H), dtype=torch.uint8, device="cuda")
if os.path.exists(out):
    os.remove(out)
for _ in range(3):
    _lib.lobra_attn_bwd(np.array(lens, np.int32), q, k, v, o, dO, lse, dq, dk, dv, wsb)
torch.cuda.synchronize()
lines = open(out).read().split("\n")
blk = [l for l in lines if l and not l.startswith("bwd")][-16:]
ts = np.array([[int(x) for x in l.split()] for l in blk], dtype=np.int64)
names = ["mma_S", "mma_dP", "mma_dV", "mma_dK", "sm_start", "sm_Pdone", "sm_dPready", "sm_dSdone",
         "mma_dO_in", "dq_empty", "dq_reds"]
base = ts[0]
print("iter " + " ".join(f"{n:>10}" for n in names) + "  period")
for t in range(32):
    row = [ts[e, t] - base[t] for e in range(len(names))]
    per = ts[0, t + 1] - ts[0, t] if t + 1 < 32 else 0
    print(f"{t:4d} " + " ".join(f"{x:10d}" for x in row) + f"  {per}")
