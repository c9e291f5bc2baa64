"""Aggregate ncu source-page warp-stall samples by CUDA source line."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = ""; agg = {}; srcs = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) < 5 or r[0] == "Line No":
        continue
    if r[0] and r[2] == "-":
        try:
            agg[(fname, int(r[0]))] = agg.get((fname, int(r[0])), 0) + int(r[4])
            srcs[(fname, int(r[0]))] = r[1][:100]
        except ValueError:
            pass
tot = sum(agg.values()) or 1
for key, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100*v/tot:5.1f}%  {key[0]}:{key[1]}  {srcs[key]}")
