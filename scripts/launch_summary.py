"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch):
per-kernel count, total/mean time and share of the profiled total."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if hdr is None:
        if "Kernel Name" in r: hdr = r
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum": continue
    name = re.sub(r"\(.*", "", d["Kernel Name"]).strip()
    name = re.sub(r"^void ", "", name)
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "")
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1.0)
    agg[name][0] += 1; agg[name][1] += v * scale
tot = sum(t for _, t in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share':>7s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:60]:60s} {n:8d} {t:12.1f} {t/n:10.2f} {100*t/tot:6.1f}%")
print(f"{'TOTAL':60s} {sum(n for n,_ in agg.values()):8d} {tot:12.1f}")
