"""Launches of the own attention forward and backward on the long-sequence case (for ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_01193_b200 import _lib  # noqa: E402

lens = [4096, 2048, 6000, 4240]
T, H = sum(lens), 32
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(T, H, 128, generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
lse = torch.empty(H, T, device="cuda")
ws = torch.empty(_lib.lobra_attn_workspace_bytes(lens, H), dtype=torch.uint8, device="cuda")
for _ in range(2):
    _lib.lobra_attn_fwd(np.array(lens, np.int32), q, k, v, o, lse, ws)
torch.cuda.synchronize()
# ... and one backward launch (lobra_attn_bwd) on the same case
dO = torch.randn(T, H, 128, generator=g, device="cuda").to(torch.bfloat16)
dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
wsb = torch.empty(_lib.lobra_attn_bwd_workspace_bytes(lens, H, H), dtype=torch.uint8, device="cuda")
for _ in range(2):
    _lib.lobra_attn_bwd(np.array(lens, np.int32), q, k, v, o, dO, lse, dq, dk, dv, wsb)
torch.cuda.synchronize()
