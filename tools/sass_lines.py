"""Attribute an ncu SASS source page (CSV) to CUDA source lines.

usage: sass_lines.py <ncu.csv from --page source --print-source sass> <nvdisasm -g -c listing>
       <mangled kernel name> [top]
Joins the per-instruction counters (warp instructions executed, thread
instructions, stall samples) with the line table nvdisasm -g prints for the same
cubin, and prints the hottest source lines."""
import csv
import re
import sys
from collections import defaultdict


def nvdis_lines(path, kernel):
    out, cur_line, inside = {}, None, False
    pat = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?);")
    for raw in open(path):
        if raw.startswith("//---------------------"):
            inside = kernel in raw
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', raw)
        if m:
            cur_line = (m.group(1).rsplit("/", 1)[-1], int(m.group(2)))
            continue
        m = pat.search(raw)
        if m:
            out[int(m.group(1), 16)] = (cur_line, m.group(2).strip())
    return out


def main():
    csv_path, dis_path, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    ia, ie, it, iss = (hdr.index("Address"), hdr.index("Instructions Executed"),
                       hdr.index("Thread Instructions Executed"),
                       hdr.index("Warp Stall Sampling (All Samples)"))
    body = [r for r in rows[hi + 1:] if len(r) > ie and r[ia].startswith("0x")]
    base = int(body[0][ia], 16)
    lines = nvdis_lines(dis_path, kernel)
    agg = defaultdict(lambda: [0, 0, 0])
    tot = [0, 0, 0]
    for r in body:
        off = int(r[ia], 16) - base
        ln = lines.get(off, (None, ""))[0]
        v = [int(r[ie] or 0), int(r[it] or 0), int(r[iss] or 0)]
        for k in range(3):
            agg[ln][k] += v[k]
            tot[k] += v[k]
    print(f"total warp instr {tot[0]:.3e}  thread instr {tot[1]:.3e}  stall samples {tot[2]}")
    src = {}

    def text(ln):
        if not ln:
            return ""
        f, n = ln
        if f not in src:
            import glob
            hits = glob.glob(f"**/{f}", recursive=True)
            src[f] = open(hits[0]).read().split("\n") if hits else []
        return src[f][n - 1].strip()[:70] if n - 1 < len(src[f]) else ""

    print("file:line                 warp_instr   %   thr/warp stall%  source")
    for ln, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        name = f"{ln[0]}:{ln[1]}" if ln else "?"
        print(f"{name:24s} {v[0]:10.3e} {100*v[0]/tot[0]:5.1f} {v[1]/max(v[0],1):6.1f} "
              f"{100*v[2]/max(tot[2],1):6.1f}  {text(ln)}")


if __name__ == "__main__":
    main()
