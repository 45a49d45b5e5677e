"""Debug helper: run one fwd/bwd case step by step with synchronisation (under gpurun)."""
import sys
import os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_01193_b200 import _lib
from workloads import synth


def run(lens, tasks, ranks, scales, d_in, d_out, what="both"):
    dev = torch.device("cuda:0")
    ts = [synth.TaskSpec(f"t{i}", 0, 0, 1, r, s) for i, (r, s) in enumerate(zip(ranks, scales))]
    wl = synth.Workload("dbg", ts, np.array(lens, np.int32), np.array(tasks, np.int32), 0)
    t = synth.layer_tensors(wl, d_in, d_out, seed=31)
    d = {k: torch.from_numpy(synth.round_bf16(v)).to(dev).to(torch.bfloat16) for k, v in t.items()}
    code = _lib.LOBRA_BF16
    ws = torch.zeros(_lib.lobra_lora_workspace_bytes(code, d_in, d_out, lens, tasks, ranks, scales), dtype=torch.uint8, device=dev)
    Hs = torch.zeros(_lib.lobra_lora_saved_bytes(code, d_in, d_out, lens, tasks, ranks, scales), dtype=torch.uint8, device=dev)
    T = wl.T
    Y = torch.empty(T, d_out, dtype=torch.bfloat16, device=dev)
    _lib.lobra_profile_enable(True)
    _lib.lobra_lora_fwd(d["X"], d["W"], d["A"], d["B"], ranks, scales, lens, tasks, Y, Hs, ws)
    torch.cuda.synchronize()
    print("fwd ok", _lib.lobra_profile_read(), flush=True)
    dX = torch.empty(T, d_in, dtype=torch.bfloat16, device=dev)
    R = sum(ranks)
    dA = torch.empty(R, d_in, dtype=torch.float32, device=dev)
    dB = torch.empty(d_out, R, dtype=torch.float32, device=dev)
    _lib.lobra_lora_bwd(d["X"], d["W"], d["A"], d["B"], ranks, scales, lens, tasks, Hs, d["dY"], dX, dA, dB, ws)
    torch.cuda.synchronize()
    print("bwd ok", _lib.lobra_profile_read(), flush=True)


if __name__ == "__main__":
    case = eval(sys.argv[1])
    run(*case)
