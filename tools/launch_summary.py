"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch):
total ms and launch count per kernel, and each kernel's share."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot, cnt, bad = {}, {}, 0
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        v = float(d["Metric Value"].replace(",", ""))
    except ValueError:
        bad += 1
        continue
    if v != v:                  # nan: a kernel node of a replayed graph
        bad += 1
        continue
    unit = d.get("Metric Unit", "nsecond")
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
    key = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
    tot[key] = tot.get(key, 0.0) + v * scale
    cnt[key] = cnt.get(key, 0) + 1
allms = sum(tot.values())
print(f"{sum(cnt.values())} launches, {allms:.2f} ms total, {bad} unparsable / untimed rows")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:40s} {cnt[k]:6d} launches {v:10.3f} ms  {100 * v / allms:5.1f} %")
