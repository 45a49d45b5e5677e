"""Per-kernel bytes / duration table from an ncu --csv launch list with dram metrics.

    python tools/skinny_table.py gpurun_out/skinny_<tag>.csv [peak_GBs]
"""
import csv
import io
import sys
from collections import defaultdict


def load(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    ker = {}
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        d = ker.setdefault(key, {"name": r["Kernel Name"].split("(")[0].replace("void ", "")})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["us"] = v / 1000.0 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1000)
        elif r["Metric Name"].startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
            d[r["Metric Name"]] = v * scale
    return [ker[k] for k in sorted(ker, key=lambda k: int(k[0]))]


def main():
    path = sys.argv[1]
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6540.8
    ks = load(path)
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    print("| # | kernel | us | DRAM MB (r+w) | GB/s | frac of HBM |")
    print("|---|---|---|---|---|---|")
    for i, k in enumerate(ks):
        b = k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
        name = k["name"].split("::")[-1][:40]
        gbs = b / (k["us"] * 1e-6) / 1e9 if k.get("us") else 0
        print(f"| {i} | {name} | {k.get('us', 0):.1f} | {b / 1e6:.1f} | {gbs:.0f} | {gbs / peak:.2f} |")
        a = agg[name.split("<")[0]]
        a[0] += 1
        a[1] += k.get("us", 0)
        a[2] += b
    print("\n| kernel class | launches | total us | total MB | GB/s | frac |")
    print("|---|---|---|---|---|---|")
    for n, (c, us, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = b / (us * 1e-6) / 1e9 if us else 0
        print(f"| {n} | {c} | {us:.1f} | {b / 1e6:.1f} | {gbs:.0f} | {gbs / peak:.2f} |")


if __name__ == "__main__":
    main()
