"""Key metrics of an ncu report (details page) as 'section | metric | value'."""
import csv
import subprocess
import sys

KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Active Warps Per SM", "Theoretical Active Warps per SM",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Executed Instructions",
        "Eligible Warps Per Scheduler", "No Eligible", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Block Limit Shared Mem", "Block Limit Registers", "Grid Size",
        "Mem Busy", "Max Bandwidth", "L1/TEX Cache Throughput", "L2 Cache Throughput")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(out.splitlines())
hdr = next(r)
for row in r:
    d = dict(zip(hdr, row))
    if d.get("Metric Name") in KEYS:
        print(f"{d['Kernel Name'][:28]:28s} | {d['Metric Name']:36s} | {d['Metric Value']:>14s} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
if len(rows) > 2:
    h, units, vals = rows[0], rows[1], rows[2:]
    for v in vals:
        d = dict(zip(h, v))
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                  "smsp__inst_executed.sum", "lts__t_bytes.sum"):
            if k in d:
                print(f"{'raw':28s} | {k:36s} | {d[k]:>14s} {units[h.index(k)]}")
