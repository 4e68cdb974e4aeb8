"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
   python scripts/launch_summary.py gpurun_out/launches.csv [top]"""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(.*", "", name)           # drop the parameter list
    name = re.sub(r"^void ", "", name)
    return name.split("::")[-1][:80]


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    tot, cnt = defaultdict(float), defaultdict(int)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for row in csv.DictReader(lines):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3}.get(row["Metric Unit"], 1e-3)
        k = short(row["Kernel Name"])
        tot[k] += float(row["Metric Value"].replace(",", "")) * scale
        cnt[k] += 1
    all_us = sum(tot.values())
    print(f"| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]:
        print(f"| {k} | {cnt[k]} | {v:.1f} | {v / cnt[k]:.1f} | {v / all_us:.1%} |")
    print(f"| total | {sum(cnt.values())} | {all_us:.1f} | | |")


if __name__ == "__main__":
    main()
