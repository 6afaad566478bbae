"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch
list: per-kernel launch count, total device time and share."""
import csv
import json
import sys

path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = {}
for r in rows[1:]:
    v = float(r[iv].replace(",", ""))
    v = {"usecond": v / 1e3, "us": v / 1e3, "nsecond": v / 1e6, "ns": v / 1e6, "msecond": v, "ms": v,
         "second": v * 1e3, "s": v * 1e3}[r[iu]]
    name = r[ik].split("(")[0][:80]
    tot.setdefault(name, []).append(v)
grand = sum(sum(v) for v in tot.values())
out = {"launch_list": path, "launches": sum(len(v) for v in tot.values()), "kernels": []}
for k, v in sorted(tot.items(), key=lambda kv: -sum(kv[1])):
    out["kernels"].append({"kernel": k, "launches": len(v), "total_ms": round(sum(v), 4),
                           "mean_ms": round(sum(v) / len(v), 4), "share": round(sum(v) / grand, 4)})
print(json.dumps(out, indent=1))
