"""The e2e leg's H2D pattern (bench.py: per micro-batch, C3's 4 X groups + 7 dY tensors from
pinned memory, largest first over 2 copy streams, double-buffered device inputs) timed
alone and with a concurrent bf16 GEMM load on another stream: does compute slow the copies?"""
import json

import torch

T = 65536
cols = [4096, 4096, 4096, 11008] + [4096] * 4 + [11008, 11008, 4096]
host = [torch.empty(T, c, dtype=torch.bfloat16, pin_memory=True) for c in cols]
dev = [[torch.empty(T, c, dtype=torch.bfloat16, device="cuda") for c in cols] for _ in range(2)]
nbytes = sum(h.numel() * 2 for h in host)
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
b = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)


def run(items, load, nstreams=2):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    comp = torch.cuda.Stream()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in ss + [comp]:
        s.wait_event(e0)
    for k in range(items):
        ld = [0] * nstreams
        for i in sorted(range(len(cols)), key=lambda i: -cols[i]):
            si = ld.index(min(ld))
            ld[si] += cols[i]
            with torch.cuda.stream(ss[si]):
                dev[k % 2][i].copy_(host[i], non_blocking=True)
        if load:
            with torch.cuda.stream(comp):
                for _ in range(load):
                    torch.matmul(a, b)
    for s in ss + [comp]:
        ev = torch.cuda.Event()
        ev.record(s)
        torch.cuda.current_stream().wait_event(ev)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


res = {"bytes_per_item": nbytes}
for load in (0, 60):
    for ns in (1, 2, 4):
        ms = run(4, load, ns)
        res[f"load{load}_s{ns}"] = {"ms": round(ms, 1), "GBps": round(4 * nbytes / ms / 1e6, 1)}
print(json.dumps(res))
