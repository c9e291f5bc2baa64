"""Summarise an ncu metrics CSV (dram bytes + duration per launch) of one
kernel family into profiles/latest_traffic.json: bytes per launch averaged
over the captured launches (bench.py's roofline `traffic`)."""
import csv, json, sys, collections
src, family, out = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
hdr = rows[0]
iid, iname, im, iv, iu = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
per = collections.defaultdict(dict)
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
for r in rows[1:]:
    per[r[iid]][r[im]] = float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
    per[r[iid]]["name"] = r[iname]
L = [v for v in per.values() if "dram__bytes_read.sum" in v]
rd = sum(v["dram__bytes_read.sum"] for v in L) / len(L)
wr = sum(v["dram__bytes_write.sum"] for v in L) / len(L)
t = sum(v.get("gpu__time_duration.sum", 0) for v in L) / len(L)
try:
    d = json.load(open(out))
except Exception:
    d = {}
d[family] = rd + wr
d[family + "_detail"] = {"launches": len(L), "dram_read_bytes_per_launch": rd, "dram_write_bytes_per_launch": wr,
                         "avg_duration_s_under_ncu": t, "kernel": L[0]["name"][:120], "source": src}
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d[family + "_detail"]))
