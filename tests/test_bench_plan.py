"""bench.py --plan-only (CPU): the N = 2/4/8 C5 deployments the stage-1 planner returns use
every GPU, and the step-0 Eq. 3 dispatch of each succeeds exactly (status 0, never the
node-budget fallback)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plan_only_deployments_and_dispatch_status():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--plan-only"], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.strip().splitlines()]
    assert [d["n_gpus"] for d in lines] == [1, 2, 4, 8]
    for d in lines:
        used = 0
        for part in d["deployment"].split("+"):
            p, rest = part.split("xTP")
            used += int(p) * int(rest.split("(")[0])
        assert used == d["n_gpus"]
        if d["n_gpus"] > 1:
            assert d["status"] == 0 and d["tokens"] == 65536 * d["n_gpus"]
