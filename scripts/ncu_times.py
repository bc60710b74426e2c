"""Summarise an `ncu --csv --metrics gpu__time_duration.sum` log: one line per
launch (kernel name, us), for quick per-kernel timing on the GPU box."""
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]      # drop ==PROF== / program output
rows = list(csv.reader(lines))
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
for r in rows[1:]:
    if len(r) <= iv:
        continue
    v = float(r[iv].replace(",", ""))
    us = v / 1000 if r[iu] == "ns" else (v * 1000 if r[iu] == "ms" else v)
    print(f"{r[ik].split('(')[0][:48]:48s} {us:9.2f} us")
