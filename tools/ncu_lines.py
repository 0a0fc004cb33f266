"""Per-source-line warp-stall samples from `ncu -i X --page source --csv --print-source cuda,sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
tot, per = 0, []
for r in rows[3:]:
    if len(r) > 5 and r[0] and r[2] == "-":
        try:
            n = int(r[4])
        except ValueError:
            continue
        per.append((n, r[0], r[1][:100]))
        tot += n
per.sort(reverse=True)
print("total samples", tot)
for n, l, s in per[:n_top]:
    print(f"{n:6d} {100 * n / max(tot, 1):5.1f}% L{l}: {s}")
