#!/usr/bin/env python
"""Key ncu metrics + top stall reasons + top SASS lines per kernel of an .ncu-rep."""
import csv
import collections
import io
import subprocess
import sys

KEEP = ['Duration', 'DRAM Throughput', 'L1/TEX Cache Throughput', 'L2 Cache Throughput',
        'Compute (SM) Throughput', 'Issue Slots Busy', 'Achieved Occupancy', 'Registers Per Thread',
        'Warp Cycles Per Issued Instruction', 'Avg. Active Threads Per Warp', 'L1/TEX Hit Rate',
        'L2 Hit Rate', 'Executed Instructions']


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, top=15):
    det = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    hdr = det[0]
    ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    iid = hdr.index("ID")
    kernels = collections.OrderedDict()
    for r in det[1:]:
        kernels.setdefault(r[iid], (r[ik], {}))[1][r[im]] = (r[iv], r[iu])
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    rh = raw[0]
    for n, (kid, (name, m)) in enumerate(kernels.items()):
        print(f"== [{kid}] {name[:110]}")
        for k in KEEP:
            if k in m:
                print(f"   {k:40s} {m[k][0]} {m[k][1]}")
        row = raw[2 + n]
        vals = dict(zip(rh, row))
        dr = vals.get("dram__bytes_read.sum"), vals.get("dram__bytes_write.sum")
        print(f"   dram read/write: {dr[0]} / {dr[1]} ({raw[1][rh.index('dram__bytes_read.sum')]})")
        st = sorted(((float(v), k.replace('smsp__pcsamp_warps_issue_stalled_', ''))
                     for k, v in vals.items()
                     if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued')
                     and v.replace('.', '').isdigit()), reverse=True)[:8]
        print("   stalls:", ", ".join(f"{k}={int(v)}" for v, k in st))
        for kk in ('l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_red.sum',
                   'l1tex__t_requests_pipe_lsu_mem_global_op_st.sum', 'l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum',
                   'l1tex__t_requests_pipe_lsu_mem_local_op_st.sum'):
            if kk in vals:
                print(f"   {kk.replace('l1tex__t_requests_pipe_lsu_mem_', '')}: {vals[kk]}")


if __name__ == "__main__":
    main(sys.argv[1])
