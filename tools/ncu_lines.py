"""Stall samples per CUDA source line of one ncu report (cuda,sass view):
    python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, fname, cur = {}, "?", None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name", "Line No"):
        continue
    if row[0]:   # a source line row: Line No, Source, then aggregated metrics
        try:
            ln = int(row[0])
        except ValueError:
            continue
        try:
            samples, execd = int(row[4] or 0), int(row[7] or 0)
        except (ValueError, IndexError):
            continue
        key = (fname, ln)
        s0, e0, src = agg.get(key, (0, 0, row[1]))
        agg[key] = (s0 + samples, max(e0, execd), row[1].strip()[:80])
tot = sum(v[0] for v in agg.values()) or 1
print(f"total stall samples {tot}")
for (f, ln), (s, e, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * s / tot:5.1f}% {e:12d}  {f}:{ln}: {src}")
