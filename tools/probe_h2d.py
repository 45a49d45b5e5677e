"""Host -> device bandwidth from pinned memory on this box (the e2e leg of bench.py is bound
by it): one large copy, and the same bytes split over 1 / 2 / 4 streams and chunk sizes."""
import json
import sys

import torch


def bw(nbytes, streams, chunk):
    src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    ss = [torch.cuda.Stream() for _ in range(streams)]
    for _ in range(2):
        best = 1e9
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for s in ss:
            s.wait_event(e0)
        off, i = 0, 0
        evs = []
        while off < nbytes:
            n = min(chunk, nbytes - off)
            with torch.cuda.stream(ss[i % streams]):
                dst[off:off + n].copy_(src[off:off + n], non_blocking=True)
            off += n
            i += 1
        for s in ss:
            ev = torch.cuda.Event()
            ev.record(s)
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return nbytes / best / 1e6


out = {}
N = 2 << 30
for streams in (1, 2, 4):
    for chunk in (64 << 20, 256 << 20, N):
        out[f"s{streams}_c{chunk >> 20}MB"] = round(bw(N, streams, chunk), 1)
print(json.dumps({"h2d_GBps": out, "device": torch.cuda.get_device_name()}))
