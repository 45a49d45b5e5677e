"""Summaries of one tools/ncu_profile.sh run (no GPU needed): copies the launch list and the
GEMM traffic CSV into profiles/, writes the per-kernel launch summary of the timed step and
updates profiles/traffic.json (bench.py's roofline.traffic).

    python tools/summarize_profiles.py r1e
"""
import collections
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def records(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    H = rows[h]
    ki, mi, vi, ii = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value"), H.index("ID")
    d = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        d.setdefault(r[ii], {"k": r[ki].split("(")[0].replace("void ", "")})[r[mi]] = float(r[vi].replace(",", ""))
    return list(d.values())


def main(tag):
    out = os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(ROOT, "profiles")
    L = records(os.path.join(out, f"launches_{tag}.csv"))
    shutil.copy(os.path.join(out, f"launches_{tag}.csv"), os.path.join(prof, f"{tag}_launches.csv"))
    L = L[len(L) // 2:]   # the timed step (warm-up step first)
    tot = collections.OrderedDict()
    for x in L:
        t = tot.setdefault(x["k"], [0, 0.0])
        t[0] += 1
        t[1] += x["gpu__time_duration.sum"] / 1000.0
    all_us = sum(v[1] for v in tot.values())
    lines = [f"# {tag}: every library launch of one bench step",
             "",
             "ncu --metrics gpu__time_duration.sum --clock-control none over `python bench.py --steps 1 --warmup 1 "
             "--profile-only` (timed step only; cold-cache, serialised: compare SHARES with bench.py's live "
             "`kernels` / `roofline.share_of_step`, not absolute times).",
             "",
             "| kernel | launches | total us | avg us | share |",
             "|---|---|---|---|---|"]
    for k, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {n} | {us:.1f} | {us / n:.1f} | {us / all_us:.3f} |")
    lines += ["", f"total {all_us:.1f} us", "", "Per launch (timed step, in order):", "",
              "| # | kernel | us |", "|---|---|---|"]
    for i, x in enumerate(L):
        lines.append(f"| {i} | {x['k']} | {x['gpu__time_duration.sum'] / 1000.0:.1f} |")
    open(os.path.join(prof, f"{tag}_launches_summary.md"), "w").write("\n".join(lines) + "\n")

    if not os.path.exists(os.path.join(out, f"gemm_traffic_{tag}.csv")):   # launch list only
        print(open(os.path.join(prof, f"{tag}_launches_summary.md")).read()[:2500])
        return
    G = records(os.path.join(out, f"gemm_traffic_{tag}.csv"))
    shutil.copy(os.path.join(out, f"gemm_traffic_{tag}.csv"), os.path.join(prof, f"{tag}_gemm_traffic.csv"))
    fwd = [x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in G if "k_gemm2<0>" in x["k"]]
    bwd = [x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in G if "k_gemm2<1>" in x["k"]]
    tj = {"k_gemm_fwd": sum(fwd) / max(len(fwd), 1), "k_gemm_bwd": sum(bwd) / max(len(bwd), 1),
          "source": f"profiles/{tag}_gemm_traffic.csv (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                    f"{len(fwd) + len(bwd)} GEMM launches of one bench step)",
          "per_launch_fwd": fwd, "per_launch_bwd": bwd}
    # bench.py looks the entry up by workload (the default bench step is C3)
    path = os.path.join(prof, "traffic.json")
    allw = json.load(open(path)) if os.path.exists(path) else {}
    allw[os.environ.get("LOBRA_TRAFFIC_WORKLOAD", "c3")] = tj
    json.dump(allw, open(path, "w"), indent=1)
    print(open(os.path.join(prof, f"{tag}_launches_summary.md")).read()[:2500])
    print(json.dumps({k: v for k, v in tj.items() if not k.startswith("per")}))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1e")
