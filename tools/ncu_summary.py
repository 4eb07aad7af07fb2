#!/usr/bin/env python
"""Summarise an `ncu --set full` report into the markdown kept under profiles/.

usage: python tools/ncu_summary.py <report.ncu-rep> [label] >> profiles/<round>_ncu.md
Also prints per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum),
the figure bench.py reports as roofline.traffic.
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput % of peak"),
    ("lts__t_sectors_op_red.sum", "L2 sectors, red"),
    ("lts__t_sectors_op_atom.sum", "L2 sectors, atom"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (achieved occupancy)"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__occupancy_limit_registers", "blocks / SM limited by registers"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
     "stall long scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
     "stall LG throttle / issue"),
    ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "stall membar / issue"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 else rep
    h, units, rows = raw(rep)
    idx = {n: i for i, n in enumerate(h)}
    print(f"## {label}\n")
    for r in rows:
        name = r[idx["Kernel Name"]].split("(")[0] if "Kernel Name" in idx else "?"
        print(f"kernel `{name[:90]}`\n")
        print("| metric | value | unit |\n|---|---|---|")
        for key, desc in METRICS:
            if key in idx:
                print(f"| {desc} (`{key}`) | {r[idx[key]]} | {units[idx[key]]} |")
        try:
            rd = to_bytes(r[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]])
            wr = to_bytes(r[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
            print(f"\nDRAM traffic per launch (read + write): {(rd + wr) / 1e9:.3f} GB\n")
            if len(sys.argv) > 3:  # profiles/traffic.json entry for bench.py roofline.traffic
                import json
                from pathlib import Path
                p = Path(sys.argv[3])
                d = json.loads(p.read_text()) if p.exists() else {}
                d[sys.argv[4] if len(sys.argv) > 4 else name] = rd + wr
                p.write_text(json.dumps(d, indent=1) + "\n")
        except (KeyError, ValueError):
            pass


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v.replace(",", "")) * scale.get(unit.strip(), 1)


if __name__ == "__main__":
    main()
