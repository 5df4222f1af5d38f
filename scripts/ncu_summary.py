"""One-screen summary of ncu --set full captures (.ncu-rep): duration, grid,
SM / DRAM / L2 throughput, occupancy, issue rate, DMMA / FP64 pipe use and the
top warp-stall reasons.   python scripts/ncu_summary.py a.ncu-rep [b.ncu-rep ...]"""
import csv, io, subprocess, sys

WANT = ["Duration", "Grid Size", "Block Size", "Registers Per Thread", "Compute (SM) Throughput",
        "Memory Throughput", "DRAM Throughput", "L2 Cache Throughput", "Achieved Occupancy",
        "Issued Ipc Active", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction"]
RAW = ["sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
       "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "dram__bytes_read.sum", "dram__bytes_write.sum"]


def rows(path, page):
    out = subprocess.run(["ncu", "-i", path, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


for path in sys.argv[1:]:
    d = rows(path, "details")
    h = d[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    print(f"== {path.split('/')[-1]}: {d[1][ki][:90]}")
    seen = set()
    for r in d[1:]:
        if len(r) > vi and r[mi] in WANT and r[mi] not in seen:
            seen.add(r[mi])
            print(f"   {r[mi]:40s} {r[vi]:>14s} {r[ui]}")
    for c in ("Grid Size", "Block Size"):
        if c in h:
            print(f"   {c:40s} {d[1][h.index(c)]:>14s}")
    rw = rows(path, "raw")
    hr, vr = rw[0], rw[2]
    stalls = []
    for k, x in zip(hr, vr):
        if k in RAW:
            print(f"   {k:70s} {x}")
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                stalls.append((float(x.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1.0
    print("   stall samples: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(stalls, reverse=True)[:5]))
