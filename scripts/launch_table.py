"""Summarise an ncu --csv launch list (gpu__time_duration.sum): python scripts/launch_table.py file.csv [skip]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr, out = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            out.append((d["Kernel Name"].split("(")[0][:60], float(d["Metric Value"]) / 1000))
out = out[skip:]
tot = sum(t for _, t in out)
for k, t in out:
    print(f"{t:9.1f} us {100 * t / tot:5.1f}%  {k}")
print(f"{tot:9.1f} us total")
