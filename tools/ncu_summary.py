"""Key metrics of every launch in an ncu --set full report (one line each):
duration, grid, SM / DRAM throughput, occupancy, IPC, DRAM bytes, top stalls.
    python tools/ncu_summary.py report.ncu-rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = {"Duration": "dur", "Grid Size": "grid", "Compute (SM) Throughput": "sm%",
        "DRAM Throughput": "dram%", "Achieved Occupancy": "occ%", "Executed Ipc Active": "ipc",
        "Registers Per Thread": "regs", "Memory Throughput": "mem"}
per = {}
for r in rows[1:]:
    d = dict(zip(hdr, r))
    key = (d["ID"], d["Kernel Name"].split("(")[0].split("::")[-1])
    m = want.get(d["Metric Name"])
    if m and (m != "mem" or d["Metric Unit"].endswith("/s")):
        per.setdefault(key, {})[m] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv",
                      "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
if rr:
    h = rr[0]
    for r in rr[2:]:
        d = dict(zip(h, r))
        key = (d.get("ID"), d.get("Kernel Name", "").split("(")[0].split("::")[-1])
        if key in per:
            try:
                b = float(d["dram__bytes_read.sum"].replace(",", "")) + \
                    float(d["dram__bytes_write.sum"].replace(",", ""))
                per[key]["dram_bytes"] = f"{b:.4g}"
            except (KeyError, ValueError):
                pass
for (i, name), m in per.items():
    print(f"[{i}] {name}: " + ", ".join(f"{k}={v}" for k, v in m.items()))
