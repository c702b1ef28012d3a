"""Top stall-sampled SASS lines of an ncu report (--set full --import-source on):
    python tools/ncu_hotspots.py report.ncu-rep [N] [context-line ...]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
isrc, iss = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
tot = sum(int(r[iss] or 0) for r in data)
print(f"{rep}: {tot} stall samples, {len(data)} SASS lines")
for i in sorted(range(len(data)), key=lambda i: -int(data[i][iss] or 0))[:top_n]:
    r = data[i]
    print(f"{i:6d} {int(r[iss]):8d} {100 * int(r[iss]) / tot:5.1f}% exec={r[ie]:>11}  {r[isrc].strip()[:90]}")
for c in sys.argv[3:]:
    a, b = (int(x) for x in c.split(":"))
    print(f"--- lines {a}..{b}")
    for i in range(a, b):
        r = data[i]
        print(f"{i:6d} {int(r[iss] or 0):8d} exec={r[ie]:>11}  {r[isrc].strip()[:100]}")
