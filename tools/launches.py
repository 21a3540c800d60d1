"""Print the per-launch device times of an ncu --metrics gpu__time_duration.sum CSV."""
import csv, sys
from collections import defaultdict

def main(path, n=14):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
    tot = defaultdict(float)
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        t = float(r[vi].replace(",", "")) / 1e3
        tot[r[ki].split("(")[0][-40:]] += t
        if n > 0:
            print(f"{t:9.1f} us  {r[ki][:48]}  {r[gi]}")
            n -= 1
    print("-- totals (us):")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{v:10.1f}  {k}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 14)
