"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel: launches, total/avg time and share.  ncu serialises launches and runs
them cold, so shares (not absolute times) compare with bench.py's `kernels`.
Usage: python tools/launch_summary.py launches.csv out.json "<source note>" """
import collections
import csv
import json
import re
import sys

src, out = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else src
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
hdr = rows[0]
iname, im, iv, iu = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
         "second": 1e6, "s": 1e6}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*$", "", r[iname]).replace("rq::(anonymous namespace)::", "")
    name = name.replace("unnamed>::", "")
    name = re.sub(r"^void ", "", name)
    us = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    agg[name][0] += 1
    agg[name][1] += us
total = sum(v[1] for v in agg.values())
by = {k: {"launches": v[0], "total_us": round(v[1], 1), "avg_us": round(v[1] / v[0], 2),
          "share": round(v[1] / total, 4)}
      for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}
json.dump({"source": note, "launches": sum(v[0] for v in agg.values()), "total_us": round(total, 1),
           "by_kernel": by}, open(out, "w"), indent=1)
print(json.dumps({k: v["share"] for k, v in list(by.items())[:8]}))
