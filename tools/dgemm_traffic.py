"""DRAM bytes per dgemm launch (and per kernel family) from an ncu launch list
with dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum of
one config-2 TNrSVD -> profiles/r02_traffic.json (bench.py's roofline.traffic).
    python tools/dgemm_traffic.py launches.csv source_note"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, per = None, collections.defaultdict(dict)
for r in rows:
    if len(r) > 5 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        per[int(d["ID"])][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        per[int(d["ID"])]["name"] = d["Kernel Name"].split("(")[0].split("::")[-1]
fam = collections.defaultdict(lambda: [0, 0.0, 0.0])
for m in per.values():
    k = "dgemm_kernel" if m["name"].startswith("dgemm_kernel") else m["name"]
    f = fam[k]
    f[0] += 1
    f[1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    f[2] += m.get("gpu__time_duration.sum", 0)
n, byt, ns = fam["dgemm_kernel"]
print(json.dumps({"kernel": "dgemm_kernel", "dram_bytes_per_launch": byt / max(n, 1),
                  "launches": n, "ncu_duration_us_per_launch": ns / max(n, 1) / 1e3,
                  "note": "average DRAM read+write bytes per dgemm launch over one config-2 "
                          "TNrSVD (all shapes); compute-bound kernel, no algorithmic-bytes "
                          "figure",
                  "families": {k: {"launches": v[0], "dram_bytes": v[1], "ms": v[2] / 1e6}
                               for k, v in sorted(fam.items(), key=lambda x: -x[1][2])[:8]},
                  "source": sys.argv[2]}, indent=1))
