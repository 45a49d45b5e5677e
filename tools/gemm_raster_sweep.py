"""Tile-order sweep of the 2-CTA GEMM on the C3 shapes with a large weight (run under gpurun).

The order is a per-shape-class tuning knob read at every launch (kernels_bf16.cu
gemm_group_m): LOBRA_GEMM_GM_NBIG for the N = 11008 GEMMs (gate/up forward, down backward)
and LOBRA_GEMM_GM_KBIG for the K = 11008 ones (down forward, gate/up backward); value g > 1:
groups of g pair-M blocks, N-major inside; 1: N-fastest; g < -1: groups of -g N blocks,
M-major inside.  Configurations are interleaved over `--rounds` rounds in ONE process so
that clock / thermal drift under the power cap hits them alike; each entry = algorithmic
TFLOP/s of the projection's forward and backward GEMMs at T = 65536 (C3 batch).

    python tools/gemm_raster_sweep.py [--nbig 16,32,-2] [--kbig 1,2,-4] [--rounds 3]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nbig", default="16,24,32,64,-2,-4")
    ap.add_argument("--kbig", default="16,1,2,3,-2,-4,-8")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--reps", type=int, default=4)
    a = ap.parse_args()
    import torch
    from paper_2509_01193_b200 import _lib
    from workloads import synth
    dev = torch.device("cuda:0")
    wl = synth.config_c3()
    T = wl.T
    R = int(wl.ranks.sum())
    code = _lib.LOBRA_BF16
    args = (wl.seq_lens, wl.seq_task, wl.ranks, wl.scales)
    bufs = {}
    for name, (d_in, d_out) in {"gate": (4096, 11008), "down": (11008, 4096)}.items():
        g = torch.Generator(device=dev).manual_seed(0)
        b = {"X": torch.randn(T, d_in, generator=g, device=dev).bfloat16(),
             "dY": torch.randn(T, d_out, generator=g, device=dev).bfloat16(),
             "W": (torch.randn(d_out, d_in, generator=g, device=dev) / d_in ** 0.5).bfloat16(),
             "A": (torch.randn(R, d_in, generator=g, device=dev) / d_in ** 0.5).bfloat16(),
             "B": (torch.randn(d_out, R, generator=g, device=dev) / 4).bfloat16(),
             "Y": torch.empty(T, d_out, dtype=torch.bfloat16, device=dev),
             "dX": torch.empty(T, d_in, dtype=torch.bfloat16, device=dev),
             "dA": torch.empty(R, d_in, dtype=torch.float32, device=dev),
             "dB": torch.empty(d_out, R, dtype=torch.float32, device=dev),
             "ws": torch.empty(_lib.lobra_lora_workspace_bytes(code, d_in, d_out, *args), dtype=torch.uint8,
                               device=dev),
             "Hs": torch.empty(_lib.lobra_lora_saved_bytes(code, d_in, d_out, *args), dtype=torch.uint8,
                               device=dev),
             "fl": 2.0 * T * d_in * d_out}
        bufs[name] = b

    def step(b):
        _lib.lobra_lora_fwd(b["X"], b["W"], b["A"], b["B"], wl.ranks, wl.scales, wl.seq_lens, wl.seq_task, b["Y"],
                            b["Hs"], b["ws"])
        _lib.lobra_lora_bwd(b["X"], b["W"], b["A"], b["B"], wl.ranks, wl.scales, wl.seq_lens, wl.seq_task, b["Hs"],
                            b["dY"], b["dX"], b["dA"], b["dB"], b["ws"])

    configs = [("NBIG", v) for v in a.nbig.split(",")] + [("KBIG", v) for v in a.kbig.split(",")]
    res = {f"{k}={v}": {"gate_fwd": [], "gate_bwd": [], "down_fwd": [], "down_bwd": []} for k, v in configs}
    for b in bufs.values():
        for _ in range(2):
            step(b)
    torch.cuda.synchronize()
    for _ in range(a.rounds):
        for k, v in configs:
            for kk in ("LOBRA_GEMM_GM_NBIG", "LOBRA_GEMM_GM_KBIG"):
                os.environ.pop(kk, None)
            os.environ["LOBRA_GEMM_GM_" + k] = v
            for name, b in bufs.items():
                step(b)
                torch.cuda.synchronize()
                _lib.lobra_profile_enable(True)
                _lib.lobra_profile_read(reset=True)
                for _ in range(a.reps):
                    step(b)
                prof = _lib.lobra_profile_read(reset=True)
                _lib.lobra_profile_enable(False)
                for d in ("fwd", "bwd"):
                    ms = prof["gemm_" + d][1] / a.reps
                    res[f"{k}={v}"][f"{name}_{d}"].append(b["fl"] / (ms / 1000) / 1e12)
    for key, r in res.items():
        print(json.dumps({"config": key, **{n: round(statistics.median(x), 1) for n, x in r.items() if x}}),
              flush=True)


if __name__ == "__main__":
    main()
