"""Where does k_rowproj's time go?  Times the forward shrink (library CUDA events, C2 batch)
under the LOBRA_DBG_RP probe bits (1 no MMA, 2 no adapter boxes, 4 no output/reduction)
and split counts, each in a fresh subprocess (the knobs are read once).  Run under gpurun."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(d_in, d_out, reps=30, bwd=False, c3=False):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2509_01193_b200 import _lib
    from workloads import synth
    dev = torch.device("cuda:0")
    wl = synth.config_c3() if c3 else synth.config_c2()
    T = wl.T
    g = torch.Generator(device=dev).manual_seed(0)
    X = torch.randn(T, d_in, generator=g, device=dev).bfloat16()
    W = (torch.randn(d_out, d_in, generator=g, device=dev) / d_in ** 0.5).bfloat16()
    R = int(wl.ranks.sum())
    A = (torch.randn(R, d_in, generator=g, device=dev) / d_in ** 0.5).bfloat16()
    B = (torch.randn(d_out, R, generator=g, device=dev) / 4).bfloat16()
    code = _lib.LOBRA_BF16
    args = (wl.seq_lens, wl.seq_task, wl.ranks, wl.scales)
    ws = torch.empty(_lib.lobra_lora_workspace_bytes(code, d_in, d_out, *args), dtype=torch.uint8, device=dev)
    Hs = torch.empty(_lib.lobra_lora_saved_bytes(code, d_in, d_out, *args), dtype=torch.uint8, device=dev)
    Y = torch.empty(T, d_out, dtype=torch.bfloat16, device=dev)
    if bwd:
        dY = torch.randn(T, d_out, generator=g, device=dev).bfloat16()
        dX = torch.empty(T, d_in, dtype=torch.bfloat16, device=dev)
        dA = torch.empty(R, d_in, dtype=torch.float32, device=dev)
        dB = torch.empty(d_out, R, dtype=torch.float32, device=dev)
        _lib.lobra_lora_fwd(X, W, A, B, wl.ranks, wl.scales, wl.seq_lens, wl.seq_task, Y, Hs, ws)
        for _ in range(reps):
            _lib.lobra_lora_bwd(X, W, A, B, wl.ranks, wl.scales, wl.seq_lens, wl.seq_task, Hs, dY, dX, dA, dB, ws)
        torch.cuda.synchronize()
        return
    for _ in range(3):
        _lib.lobra_lora_fwd(X, W, A, B, wl.ranks, wl.scales, wl.seq_lens, wl.seq_task, Y, Hs, ws)
    torch.cuda.synchronize()
    _lib.lobra_profile_enable(True)
    _lib.lobra_profile_read(reset=True)
    for _ in range(reps):
        _lib.lobra_lora_fwd(X, W, A, B, wl.ranks, wl.scales, wl.seq_lens, wl.seq_task, Y, Hs, ws)
    prof = _lib.lobra_profile_read(reset=True)
    n, ms = prof["rowproj"]
    us = 1000 * ms / n
    print(json.dumps({"us": us, "GBps": T * d_in * 2 / (us * 1e-6) / 1e9}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] in ("child", "childb", "childb3"):
        child(int(sys.argv[2]), int(sys.argv[3]), reps=6 if sys.argv[1] != "child" else 30,
              bwd=sys.argv[1] != "child", c3=sys.argv[1] == "childb3")
        sys.exit(0)
    combos = [{"LOBRA_SHRINK": "0"}, {"LOBRA_SHRINK": "1"}]
    if os.environ.get("PROBE_ALL"):
        for dbg in ("1", "2", "3", "4", "7"):
            combos.append({"LOBRA_SHRINK": "0", "LOBRA_DBG_RP": dbg})
    for shape in ((4096, 4096), (11008, 4096)):
        for c in combos:
            env = dict(os.environ, **c)
            out = subprocess.run([sys.executable, __file__, "child", str(shape[0]), str(shape[1])], env=env,
                                 capture_output=True, text=True, timeout=300)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
            print(f"in={shape[0]:6d} {json.dumps(c):70s} {line}", flush=True)
