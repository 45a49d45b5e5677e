"""Per-phase clock64 trace of CTA 0 of the attention forward (LOBRA_TRACE_ATTN=<file>): one
4096-token sequence, CTA 0 = its last query tile (32 key tiles).  SM cycles relative to
the first S issue."""
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
q, k, v = (torch.randn(T, H, 128, generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
lse = torch.empty(H, T, device="cuda")
ws = torch.empty(_lib.lobra_attn_workspace_bytes(lens, H), dtype=torch.uint8, device="cuda")
if os.path.exists(out):
    os.remove(out)
for _ in range(3):
    _lib.lobra_attn_fwd(np.array(lens, np.int32), q, k, v, o, lse, ws)
torch.cuda.synchronize()
lines = [l for l in open(out).read().split("\n") if l and not l.startswith("fwd")][-16:]
ts = np.array([[int(x) for x in l.split()] for l in lines], dtype=np.int64)
names = ["prod_kv", "mma_S", "mma_PV", "sm_S", "sm_max", "sm_ofull", "sm_Pdone"]
base = ts[1, 0]
print("tile " + " ".join(f"{n:>9}" for n in names) + "  S-period")
for t in range(32):
    print(f"{t:4d} " + " ".join(f"{ts[e, t] - base:9d}" for e in range(len(names))) +
          f"  {ts[1, t + 1] - ts[1, t] if t + 1 < 32 else 0}")
