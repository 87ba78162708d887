"""Key metrics of an ncu report (details page): duration, DRAM bytes/throughput, occupancy, IPC, stalls."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy", "Achieved Active Warps Per SM",
        "Block Limit Registers", "Block Limit Shared Mem", "Executed Instructions", "L2 Hit Rate", "Waves Per SM",
        "Warp Cycles Per Issued Instruction", "Max Active Clusters", "Grid Size"]
seen = set()
for r in rows[1:]:
    name = r[ix["Metric Name"]]
    key = (r[ix["ID"]], name)
    if name in want and key not in seen:
        seen.add(key)
        print(f"[{r[ix['ID']]}] {name:40s} {r[ix['Metric Value']]:>16s} {r[ix['Metric Unit']]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h = rr[0]
for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "lts__t_bytes.sum"):
    if name in h:
        i = h.index(name)
        for row in rr[2:]:
            print(f"{name:40s} {row[i]:>16s} {rr[1][i]}")
