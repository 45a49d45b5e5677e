"""Step-time sensitivity to launch plumbing (run under gpurun): the C2 layer step on one fixed
batch, uninstrumented, under env variants (each in a fresh process: the knobs are read once).
  LOBRA_META_CACHE=1  skip the per-call metadata H2D when the device copy is identical
  LOBRA_NO_PDL=1      no programmatic dependent launch"""
import json
import numpy as np
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(steps=30):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2509_01193_b200 import _lib
    from paper_2509_01193_b200.layer import LLAMA2_7B, LoraLayer
    from workloads import synth
    dev = torch.device("cuda:0")
    _lib.load()
    tasks = synth.c2_tasks()
    layer = LoraLayer(LLAMA2_7B, [t.rank for t in tasks], [t.scale for t in tasks], dev, torch.bfloat16, 1, 0,
                      None, seed=1234)
    io = layer.alloc_io(16384, seed=99)
    wl = synth.config_c2()
    lens, tsk, T = wl.seq_lens.astype(np.int32), wl.seq_task.astype(np.int32), wl.T

    def step():
        layer.forward(lens, tsk, io, T)
        layer.backward(lens, tsk, io, T, accumulate_dadb=False)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"ms_per_step": e0.elapsed_time(e1) / steps}))


if __name__ == "__main__":
    import numpy as np   # noqa: F401  (child uses it)
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
        sys.exit(0)
    for env in ({}, {"LOBRA_META_CACHE": "1"}, {"LOBRA_NO_PDL": "1"}, {}, {"LOBRA_META_CACHE": "1"}):
        out = subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, **env),
                             capture_output=True, text=True, timeout=600)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:]
        print(json.dumps(env), line, flush=True)
