"""Aggregate an ncu source page (cuda,sass) by CUDA source line: instructions executed and stall samples."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
data = []
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        i_ie = hdr.index("Instructions Executed")
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= i_ie or not r[0]:
        continue
    try:
        data.append((int(r[i_ie]), int(r[i_s]), r[0], r[1][:100]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
ts = sum(d[1] for d in data) or 1
print("total warp-instructions", tot, "stall samples", ts)
key = 1 if "--stall" in sys.argv else 0
for d in sorted(data, key=lambda d: -d[key])[:n]:
    print(f"{d[0]:>11} {100*d[0]/tot:5.1f}%  stall {100*d[1]/ts:5.1f}%  L{d[2]:>4} {d[3]}")
