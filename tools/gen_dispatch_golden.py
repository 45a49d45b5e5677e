"""Writes tests/golden/dispatch_c5.json: the ORACLE's Eq. 3 dispatch of C5-scale steps.

Calls only oracle/ and workloads/ (test infrastructure): every expected value in the
fixture comes from oracle.dispatch.dispatch (HiGHS path with integer-certified answers,
DESIGN.md "HiGHS"), never from the CUDA/C++ library.  The instances follow SURVEY §8(d) C5:
one step's global batch of C3's 16 tasks (dataset-table batch sizes for the 12 tasks, 64 for
the 4 clones: B ~ 1952 sequences), grid 256 / 16384, R = 16, integer per-sequence costs
round((s + s^2/16384) / (tp * 0.85^log2 tp) / 32) (App. D shape, reading Q15), and the
deployments
    G2  : TP1 x4 (M 8192) + TP2 x2 (M 16384)                         8 GPUs
    G3  : TP1 x2 (M 8192) + TP2 x1 + TP4 x1 (M 16384)                8 GPUs
    G3p : TP1 x4 (M 8192) + TP2 x2 + TP4 x1 (M 16384)               12 GPUs
    G4  : TP1 x2 (M 8192) + TP2 x1 + TP4 x1 + TP8 x1 (M 16384)      16 GPUs
with seeds 100..104.  The fixture stores d, t_hat and a SHA-256 of the per-sequence
outputs (bucket, replica, chunk, packing order, replica costs) for chunking = 1.

    python tools/gen_dispatch_golden.py            # ~5-10 min (the oracle's MILPs)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import dispatch as D  # noqa: E402
from workloads import synth  # noqa: E402

DEPLOYMENTS = {
    "G2": [(1, 4, 8192), (2, 2, 16384)],
    "G3": [(1, 2, 8192), (2, 1, 16384), (4, 1, 16384)],
    "G3p": [(1, 4, 8192), (2, 2, 16384), (4, 1, 16384)],
    "G4": [(1, 2, 8192), (2, 1, 16384), (4, 1, 16384), (8, 1, 16384)],
}
SEEDS = list(range(100, 105))
STEP, GMAX, R, UNIT = 256, 16384, 16, 32


def cost_table(groups):
    out = []
    for g in groups:
        eff = g.tp * (0.85 ** np.log2(g.tp))
        out.append([max(1, int(round(((k + 1) * STEP + ((k + 1) * STEP) ** 2 / 16384) / eff / UNIT)))
                    for k in range(GMAX // STEP)])
    return out


def batch(seed):
    tasks = synth.c3_tasks()
    return synth.sample_batch(tasks, seed=seed, l_max=GMAX,
                              per_task=[t.batch_size for t in tasks[:12]] + [64] * 4)


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes())
    return h.hexdigest()


def main():
    cases = []
    for name, dep in DEPLOYMENTS.items():
        groups = [D.Group(*g) for g in dep]
        cost = cost_table(groups)
        for seed in SEEDS:
            wl = batch(seed)
            t0 = time.time()
            res = D.dispatch(groups, cost, wl.seq_lens, wl.seq_task, STEP, GMAX, R, mode=0, chunking=1)
            dt = time.time() - t0
            cases.append({"name": name, "deployment": dep, "seed": seed, "num_seqs": int(len(wl.seq_lens)),
                          "boundaries": res.boundaries, "d": res.d.tolist(), "t_hat": res.t_hat,
                          "sha256": digest(res.seq_bucket, res.seq_replica, res.seq_chunk, res.pack_order,
                                           res.replica_cost),
                          "oracle_seconds": round(dt, 2)})
            print(name, seed, res.t_hat, f"{dt:.1f}s", flush=True)
    out = {"source": "tools/gen_dispatch_golden.py (oracle.dispatch only)",
           "grid_step": STEP, "grid_max": GMAX, "R": R, "cost_unit": UNIT, "chunking": 1,
           "cases": cases}
    with open(os.path.join(ROOT, "tests", "golden", "dispatch_c5.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
