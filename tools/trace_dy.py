"""Per-CTA time of the backward dY pass (k_dypass) on the bench workload, with each CTA's
entry ranges (LOBRA_TRACE_DY=<file> makes the library write one JSON line per launch): the
spread of CTA durations and a least-squares split of a CTA's time into per-entry and
per-segment costs (run under gpurun after one bench step)."""
import json
import sys

import numpy as np

recs = [json.loads(l) for l in open(sys.argv[1])]
print(f"{len(recs)} launches")
for r in recs:
    ctas = r["cta"]
    d = np.array([(c[1] - c[0]) / 1e3 for c in ctas])           # us
    start = np.array([c[0] for c in ctas], np.float64)
    end = np.array([c[1] for c in ctas], np.float64)
    ent = np.array([sum(u[3] - u[2] for u in c[3]) for c in ctas], np.float64)
    seg = np.array([len(c[3]) for c in ctas], np.float64)
    r64 = np.array([sum((u[3] - u[2]) * (r["ranks"][u[0]] > 32) for u in c[3]) for c in ctas], np.float64)
    A = np.stack([ent, seg, r64, np.ones_like(ent)], 1)
    coef, *_ = np.linalg.lstsq(A, d, rcond=None)
    pred = A @ coef
    print(f"width {r['width']:5d} qp {r['qp']} ctas {len(ctas)}: span {(end.max() - start.min()) / 1e3:7.1f} us, "
          f"CTA time min/mean/max {d.min():6.1f}/{d.mean():6.1f}/{d.max():6.1f} us, start spread "
          f"{(start.max() - start.min()) / 1e3:5.1f} us; entries/CTA {ent.min():.0f}-{ent.max():.0f}, "
          f"segments/CTA {seg.min():.0f}-{seg.max():.0f}; fit us = {coef[0]:.2f}*entry + {coef[1]:.2f}*segment "
          f"+ {coef[2]:.2f}*rank>32 entry + {coef[3]:.1f} (rms {np.sqrt(np.mean((pred - d) ** 2)):.1f})")
