"""Micro-benchmark of the per-projection kernels on the C2 shapes (run under gpurun).
Prints per-kernel-class average device time and the algorithmic HBM GB/s of the
memory-bound classes (rowproj reads T*K*2 bytes, segred reads T*width*2 bytes)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_01193_b200 import _lib
from workloads import synth


def run(d_in, d_out, reps=20):
    dev = torch.device("cuda:0")
    wl = synth.config_c2()
    T = wl.T
    g = torch.Generator(device=dev).manual_seed(0)
    X = torch.randn(T, d_in, generator=g, device=dev).bfloat16()
    dY = torch.randn(T, d_out, generator=g, device=dev).bfloat16()
    W = (torch.randn(d_out, d_in, generator=g, device=dev) / d_in ** 0.5).bfloat16()
    R = int(wl.ranks.sum())
    A = (torch.randn(R, d_in, generator=g, device=dev) / d_in ** 0.5).bfloat16()
    B = (torch.randn(d_out, R, generator=g, device=dev) / 4).bfloat16()
    code = _lib.LOBRA_BF16
    args = (wl.seq_lens, wl.seq_task, wl.ranks, wl.scales)
    ws = torch.empty(_lib.lobra_lora_workspace_bytes(code, d_in, d_out, *args), dtype=torch.uint8, device=dev)
    Hs = torch.empty(_lib.lobra_lora_saved_bytes(code, d_in, d_out, *args), dtype=torch.uint8, device=dev)
    Y = torch.empty(T, d_out, dtype=torch.bfloat16, device=dev)
    dX = torch.empty(T, d_in, dtype=torch.bfloat16, device=dev)
    dA = torch.empty(R, d_in, dtype=torch.float32, device=dev)
    dB = torch.empty(d_out, R, dtype=torch.float32, device=dev)

    def step():
        _lib.lobra_lora_fwd(X, W, A, B, wl.ranks, wl.scales, wl.seq_lens, wl.seq_task, Y, Hs, ws)
        _lib.lobra_lora_bwd(X, W, A, B, wl.ranks, wl.scales, wl.seq_lens, wl.seq_task, Hs, dY, dX, dA, dB, ws)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    _lib.lobra_profile_enable(True)
    _lib.lobra_profile_read(reset=True)
    for _ in range(reps):
        step()
    prof = _lib.lobra_profile_read(reset=True)
    _lib.lobra_profile_enable(False)
    out = {}
    for k, (n, ms) in prof.items():
        if n:
            out[k] = {"launches": n, "us_avg": 1000 * ms / n}
    # rowproj: fwd reads X (T*in*2), bwd reads dY (T*out*2)
    rp_bytes = (T * d_in * 2 + T * d_out * 2) * reps
    sr_bytes = (T * d_in * 2 + T * d_out * 2) * reps
    if "rowproj" in prof:
        out["rowproj"]["GBps"] = rp_bytes / (prof["rowproj"][1] / 1000) / 1e9
    if "segred" in prof:
        out["segred"]["GBps"] = sr_bytes / (prof["segred"][1] / 1000) / 1e9
    fl = 2.0 * T * d_in * d_out * reps
    for k in ("gemm_fwd", "gemm_bwd"):
        if k in prof:
            out[k]["TFLOPs"] = fl / (prof[k][1] / 1000) / 1e12
    return out


if __name__ == "__main__":
    torch.cuda.set_device(0)
    res = {}
    for name, (i, o) in {"q": (4096, 4096), "gate": (4096, 11008), "down": (11008, 4096)}.items():
        res[name] = run(i, o)
    print(json.dumps(res))
