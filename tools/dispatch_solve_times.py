"""Solve time of lobra_dispatch (mode 0, exact Eq. 3) on the C5-scale fixture instances
(tests/golden/dispatch_c5.json) -- median of 3 calls each, one host core.

    python tools/dispatch_solve_times.py > profiles/r2_dispatch_solve_times.md
"""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2509_01193_b200 import _lib  # noqa: E402
from oracle import dispatch as D  # noqa: E402
from test_dispatch_cpp import _c5_cost  # noqa: E402
from workloads import synth  # noqa: E402

C5 = json.load(open(os.path.join(ROOT, "tests", "golden", "dispatch_c5.json")))
print("# lobra_dispatch solve times, C5-scale steps (B ~ 1952, R = 16, grid 256/16384)\n")
print("Every result is bit-exact vs the oracle fixture (tests/test_dispatch_cpp.py). "
      "`oracle s` = the oracle's HiGHS path on the same instance (fixture generation).\n")
print("| deployment | groups | seed | t_hat | B&B nodes | C++ ms (median of 3) | oracle s |")
print("|---|---|---|---|---|---|---|")
per = {}
for case in C5["cases"]:
    groups = [D.Group(*g) for g in case["deployment"]]
    cost = _c5_cost(groups, C5["cost_unit"])
    tasks = synth.c3_tasks()
    wl = synth.sample_batch(tasks, seed=case["seed"], l_max=16384,
                            per_task=[t.batch_size for t in tasks[:12]] + [64] * 4)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        got = _lib.lobra_dispatch([g.tp for g in groups], [g.replicas for g in groups],
                                  [g.max_tokens for g in groups], cost, wl.seq_lens, wl.seq_task,
                                  C5["grid_step"], C5["grid_max"], C5["R"], 0, chunking=C5["chunking"])
        ts.append(1000 * (time.perf_counter() - t0))
    assert got["d"].tolist() == case["d"]
    ms = statistics.median(ts)
    per.setdefault(case["name"], []).append(ms)
    dep = "+".join(f"{p}xTP{tp}" for tp, p, _ in case["deployment"])
    print(f"| {case['name']} {dep} | {len(groups)} | {case['seed']} | {case['t_hat']} | "
          f"{got['nodes'] if len(groups) >= 3 else '(2-group DP)'} | {ms:.1f} | {case['oracle_seconds']} |")
print()
for k, v in per.items():
    print(f"* {k}: median {statistics.median(v):.1f} ms, max {max(v):.1f} ms")
