#!/usr/bin/env python
"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv
--log-file X.csv ...`) into the per-kernel markdown table kept under profiles/.

usage: python tools/launch_summary.py <launches.csv> "<command line>" > profiles/<name>.md
"""
import csv
import io
import re
import sys
from collections import defaultdict


def main():
    path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        m = re.search(r"(k_[A-Za-z0-9_]+)", name)
        key = m.group(1) if m else name[:40]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ms = v / 1e6 if unit in ("nsecond", "ns") else (v / 1e3 if unit in ("usecond", "us") else v)
        per[key][0] += 1
        per[key][1] += ms
    total = sum(v[1] for v in per.values())
    print(f"# launch list — `{cmd}`\n")
    print("Cold-cache, serialised per-launch times (ncu replays each kernel): compare "
          "shares, not absolutes.\n")
    print("| kernel | launches | total ms | mean ms | share |\n|---|---|---|---|---|")
    for k, (n, ms) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {ms:.3f} | {ms / n:.4f} | {100 * ms / total:.1f}% |")
    print(f"| total | {sum(v[0] for v in per.values())} | {total:.3f} | | |")


if __name__ == "__main__":
    main()
