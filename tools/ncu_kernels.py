#!/usr/bin/env python
"""Per-kernel limiter counters from an `ncu --set full` capture of the bench, as
the JSON bench.py folds into its roofline object (profiles/kernels.json).

usage: python tools/ncu_kernels.py <report.ncu-rep> <out.json> [source note]
For each captured launch of K0 (k_map_forward_rec -> "map_forward") and K2
(k_map_backward_q -> "map_backward"): DRAM bytes (read + write), duration, and
the counters that name the real limiter (L1 / L2 throughput, issue active,
warps active, warp instructions, active threads per warp, registers).
"""
import csv
import io
import json
import subprocess
import sys

SLOTS = {"k_map_forward_rec": "map_forward", "k_map_backward_q": "map_backward",
         "k_rmsprop_blocks": "rmsprop", "k_pose_group_u": "pose_gn"}
METRICS = {
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__time_duration.sum": "duration",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_warp_inst",
    "launch__registers_per_thread": "registers",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "lts__t_sectors_op_red.sum": "l2_red_sectors",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, body = rows[0], rows[1], rows[2:]
    ix = {n: i for i, n in enumerate(hdr)}
    res = {"_source": f"{rep}" + (f" ({sys.argv[3]})" if len(sys.argv) > 3 else "")}
    for r in body:
        name = r[ix["Kernel Name"]]
        slot = next((v for k, v in SLOTS.items() if k + "<" in name or k + "(" in name), None)
        if slot is None:
            continue
        d = {}
        for key, short in METRICS.items():
            if key not in ix or not r[ix[key]]:
                continue
            v = float(r[ix[key]].replace(",", ""))
            u = units[ix[key]].strip()
            if short.startswith("dram_read") or short.startswith("dram_write"):
                v *= SCALE.get(u, 1)
            elif short == "duration":
                v *= SCALE.get(u, 1)  # -> ms
            d[short] = v
        d["dram_bytes"] = d.get("dram_read", 0.0) + d.get("dram_write", 0.0)
        d["duration_ms"] = d.pop("duration", None)
        res[slot] = d
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
        f.write("\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
