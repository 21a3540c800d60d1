"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch):
total time and count per kernel, largest first."""
import collections
import csv
import io
import sys


def main(path, top=15):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in csv.DictReader(io.StringIO("\n".join(lines[start:]))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += float(r["Metric Value"].replace(",", ""))
    tot = sum(t for _, t in agg.values())
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{t / 1e3:10.1f} us {100 * t / tot:5.1f}%  {n:4d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
