"""Summarise an ncu --csv launch list (gpu__time_duration.sum and, when
captured, dram bytes) per launch: python tools/launch_table.py FILE.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
k = collections.OrderedDict()
for d in data:
    k.setdefault((d["ID"], d["Kernel Name"]), {})[d["Metric Name"]] = float(
        d["Metric Value"].replace(",", ""))
tot = 0.0
for (i, n), m in k.items():
    us = m.get("gpu__time_duration.sum", 0) / 1e3
    tot += us
    rd = m.get("dram__bytes_read.sum", 0) / 1e9
    wr = m.get("dram__bytes_write.sum", 0) / 1e9
    print(f"{i:>4} {n.split('(')[0][-40:]:<40} {us:9.1f} us  dram rd {rd:6.2f} GB  wr {wr:6.2f} GB")
print(f"total {tot / 1e3:.2f} ms over {len(k)} launches")
