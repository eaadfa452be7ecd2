"""Print the key ncu metrics + rule messages of every launch in a report (development aid)."""
import csv
import io
import subprocess
import sys

KEYS = ("Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Mem Pipes Busy", "Achieved Occupancy",
        "Warp Cycles Per Issued Instruction", "Issued Instructions", "Registers Per Thread", "Grid Size",
        "Dynamic Shared Memory Per Block", "No Eligible", "Active Warps Per Scheduler", "L2 Hit Rate", "L1/TEX Hit Rate")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))[1:]
cur = None
for r in rows:
    if r[0] != cur:
        cur = r[0]
        print(f"== launch {cur}: {r[4][:70]}")
    if r[12] in KEYS:
        print(f"   {r[12][:40]:40s} {r[14]} {r[13]}")
    elif len(r) > 17 and r[17] and ("-v" in sys.argv):
        print(f"   * {r[17][:400]}")
