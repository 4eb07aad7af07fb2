#!/usr/bin/env python
"""SASS excerpts of a kernel from an `nvdisasm -g -c` listing, by opcode.

usage: sass_excerpt.py <listing> <mangled-name-fragment> <opcode-regex> [max]
Prints the instruction count of the kernel and every instruction matching the
regex with the source line the line table gives it (the evidence that e.g. the
corner gathers are LDG.E.128 and the scatter is RED.E.ADD.F32x4)."""
import re
import sys


def main():
    path, frag, pat = sys.argv[1], sys.argv[2], re.compile(sys.argv[3])
    cap = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    inside, cur, n, hits = False, None, 0, []
    for raw in open(path):
        if raw.startswith("//---------------------"):
            inside = frag in raw
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', raw)
        if m:
            cur = f"{m.group(1).rsplit('/', 1)[-1]}:{m.group(2)}"
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", raw)
        if m:
            n += 1
            if pat.search(m.group(2)):
                hits.append(f"/*{m.group(1)}*/ {m.group(2).strip():60s} // {cur}")
    print(f"{len(hits)} of {n} instructions match /{pat.pattern}/")
    for h in hits[:cap]:
        print("  ", h)
    if len(hits) > cap:
        print(f"   ... {len(hits) - cap} more")


if __name__ == "__main__":
    main()
