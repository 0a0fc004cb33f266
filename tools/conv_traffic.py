"""Whole-conversion DRAM bytes per conversion from an ncu launch list
(dram__bytes_read.sum + dram__bytes_write.sum over the conversion kernels,
divided by the number of conversions in the capture) -> JSON for bench.py.
    python tools/conv_traffic.py launches.csv n_conversions source_note > profiles/r02_conv_traffic.json"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
nconv = int(sys.argv[2])
hdr, per = None, collections.defaultdict(dict)
for r in rows:
    if len(r) > 5 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        per[int(d["ID"])][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        per[int(d["ID"])]["name"] = d["Kernel Name"].split("(")[0]
tot = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in per.values())
dur = sum(m.get("gpu__time_duration.sum", 0) for m in per.values())
print(json.dumps({"kernel": "whole conversion (" + ", ".join(sorted({m["name"].split("::")[-1] for m in per.values()})) + ")",
                  "dram_bytes_per_step": tot / nconv, "ncu_duration_ms": dur / nconv / 1e6,
                  "source": sys.argv[3]}, indent=1))
