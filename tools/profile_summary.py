"""Summarise ncu outputs of a round into profiles/ (tracked): the launch list of the bench command
and the full capture of the dominant kernel.

    python tools/profile_summary.py <tag> <launches.csv> <full.ncu-rep> [bench.json]
"""
import collections
import csv
import json
import os
import subprocess
import sys

tag, launches, rep = sys.argv[1], sys.argv[2], sys.argv[3]
bench = sys.argv[4] if len(sys.argv) > 4 else None
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(root, "profiles")
os.makedirs(out, exist_ok=True)

# 1. launch list: per kernel count, mean duration, share of the captured launches
rows = [r for r in csv.reader(open(launches)) if len(r) > 5]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
per = collections.defaultdict(list)
for r in rows[1:]:
    if r[ix["Metric Name"]] == "gpu__time_duration.sum":
        per[r[ix["Kernel Name"]]].append(float(r[ix["Metric Value"]]))
tot = sum(sum(v) for v in per.values())
launch_summary = {k: {"launches": len(v), "mean_us": sum(v) / len(v) / 1e3, "share": sum(v) / tot} for k, v in per.items()}

# 2. full capture: the metrics the roofline uses
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, units, vals = rr[0], rr[1], rr[2]
want = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
full = {}
for name in want:
    if name in h:
        i = h.index(name)
        full[name] = {"value": vals[i], "unit": units[i]}


def num(name, scale):
    u = full[name]["unit"].lower()
    v = float(full[name]["value"].replace(",", ""))
    f = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "nsecond": 1e-9, "msecond": 1e-3}.get(u, 1)
    return v * f / scale


traffic = num("dram__bytes_read.sum", 1) + num("dram__bytes_write.sum", 1)
summary = {"tag": tag, "launch_list": launch_summary, "full_capture": full, "dram_traffic_bytes_per_launch": traffic}
if bench:
    summary["bench"] = json.loads(open(bench).read().strip().splitlines()[-1])
with open(os.path.join(out, f"{tag}_ncu_summary.json"), "w") as fh:
    json.dump(summary, fh, indent=1)
print(json.dumps({"traffic": traffic, "launch_list": launch_summary}, indent=1))
