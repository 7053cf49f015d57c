"""Per-kernel share of device time from an ncu launch list (--metrics gpu__time_duration.sum --csv).
    python scripts/launch_list_summary.py launches.csv out.json "<how it was captured>" """
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
tot, n = collections.Counter(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    k = r[ik].split("(")[0]
    tot[k] += float(r[iv].replace(",", "")) * scale[r[iu]]
    n[k] += 1
T = sum(tot.values())
out = {"source": sys.argv[3] if len(sys.argv) > 3 else sys.argv[1],
       "kernels": [{"kernel": k, "launches": n[k], "total_us": tot[k], "mean_us": tot[k] / n[k],
                    "share": tot[k] / T} for k, _ in tot.most_common()]}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
