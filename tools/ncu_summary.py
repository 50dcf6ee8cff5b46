import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
ik = h.index("Kernel Name"); isec = h.index("Section Name"); im = h.index("Metric Name"); iu = h.index("Metric Unit"); iv = h.index("Metric Value")
want = {"Duration", "Elapsed Cycles", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Issued Warp Per Scheduler", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Theoretical Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block",
        "Active Warps Per Scheduler", "Eligible Warps Per Scheduler", "Issue Slots Busy"}
cur = None
for row in r[1:]:
    if row[ik] != cur:
        cur = row[ik]; print("==", cur[:90])
    if row[im] in want:
        print(f"   {row[im]:40s} {row[iv]:>14s} {row[iu]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hh = rr[0]
for row in rr[2:]:
    st = sorted(((float(v), a.replace("smsp__pcsamp_warps_issue_stalled_", "")) for a, v in zip(hh, row)
                 if a.startswith("smsp__pcsamp_warps_issue_stalled") and not a.endswith("not_issued") and v.replace('.', '', 1).isdigit()), reverse=True)[:7]
    dr = [(a, v) for a, v in zip(hh, row) if a in ("dram__bytes_read.sum", "dram__bytes_write.sum")]
    print("  stalls:", ", ".join(f"{n}={int(v)}" for v, n in st), "|", dr)
