#!/usr/bin/env python
"""List a kernel's local-memory stores/loads (STL/LDL) with their stack offsets and
source lines, and flag loads from offsets the kernel never stores to.

usage: python tools/sass_spills.py <lib.so> <cubin name, e.g. vrf_track> <kernel substring>
(r02: found ptxas spilling k_pose_group_u at 4 CTAs/SM with LDL.LU from [R1+0x60]
and [R1+0x68] and no STL to either slot, profiles/r02_pose_minb4_spill_bug.md)."""
import re
import subprocess
import sys
import tempfile
from pathlib import Path


def main(lib, cub, kern):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(Path(lib).resolve())], cwd=d,
                       check=True, capture_output=True)
        cubin = next(Path(d).glob(f"{cub}*.cubin"))
        sass = subprocess.run(["nvdisasm", "-g", "-c", str(cubin)], check=True,
                              capture_output=True, text=True).stdout.split("\n")
    inside, line, stores, loads = False, None, set(), []
    for raw in sass:
        if raw.startswith("//---------------------"):
            inside = kern in raw
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', raw)
        if m:
            line = f"{m.group(1).rsplit('/', 1)[-1]}:{m.group(2)}"
            continue
        m = re.search(r"\b(STL|LDL)(\.[A-Z0-9.]+)?\s+(.*?);", raw)
        if not m:
            continue
        off = re.search(r"\[R1(?:\+0x([0-9a-f]+))?\]", m.group(3))
        o = int(off.group(1) or "0", 16) if off else None
        print(f"{line:28s} {m.group(1)}{m.group(2) or ''} {m.group(3)}")
        if m.group(1) == "STL":
            stores.add(o)
        elif o is not None:
            loads.append((o, line))
    bad = [(o, ln) for o, ln in loads if o not in stores and None not in stores]
    print("loads from never-stored R1 offsets:", bad if bad else "none")


if __name__ == "__main__":
    main(*sys.argv[1:4])
