"""Aggregate ncu source-page executed instructions + stall samples per CUDA line."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = ""; agg = {}; srcs = {}; hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] and r[2] == "-":
        try:
            key = (fname, int(r[0]))
            ie = hdr.index("Instructions Executed")
            v = agg.setdefault(key, [0, 0])
            v[0] += int(r[4]); v[1] += int(r[ie])
            srcs[key] = r[1][:90]
        except (ValueError, IndexError):
            pass
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total warp-inst executed {ti}")
for key, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"inst {100*v[1]/ti:5.1f}%  stall {100*v[0]/ts:5.1f}%  {key[0]}:{key[1]}  {srcs[key]}")
