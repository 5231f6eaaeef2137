"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel name: launches, total ms, share.  python tools/launch_table.py FILE.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].replace("void ", "").replace("(anonymous namespace)::", "")
        base = name.split("(")[0].split("<")[0]
        name = base.split("::")[-1] + ("<...>" if "<" in name.split("(")[0] else "")
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(d["Metric Unit"], 1e-6)
        agg[name][0] += 1
        agg[name][1] += v
tot = sum(x[1] for x in agg.values())
print(f"{'kernel':36s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:36s} {n:8d} {ms:10.3f} {100 * ms / tot:6.1f}%")
print(f"{'total':36s} {sum(x[0] for x in agg.values()):8d} {tot:10.3f}")
