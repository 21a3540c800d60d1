"""Instruction / stall breakdown of one kernel of an ncu report by SASS address
region, plus the hottest instructions with their dominant stall reasons.

usage: ncu_regions.py REPORT [region_bytes=0x400] [blocks=1] [top=25]"""
import collections
import csv
import io
import subprocess
import sys

REASONS = ["stall_wait", "stall_short_sb", "stall_long_sb", "stall_math", "stall_mio", "stall_barrier",
           "stall_branch_resolving", "stall_not_selected", "stall_selected", "stall_dispatch", "stall_lg",
           "stall_no_inst"]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[h]
    col = {c: hdr.index(c) for c in ["Source", "Instructions Executed", "Warp Stall Sampling (All Samples)"] + REASONS}
    data = []
    for r in rows[h + 1:]:
        try:
            a = int(r[0], 16)
        except (ValueError, IndexError):
            continue
        f = lambda c: float(r[col[c]] or 0)
        data.append(dict(addr=a, src=r[col["Source"]], inst=f("Instructions Executed"),
                         samp=f("Warp Stall Sampling (All Samples)"), **{k: f(k) for k in REASONS}))
    return data


def main(path, region=0x400, blocks=1, top=25):
    d = load(path)
    base = d[0]["addr"]
    ti = sum(x["inst"] for x in d) or 1
    ts = sum(x["samp"] for x in d) or 1
    print(f"warp instructions {ti:.4g} ({ti / blocks:.1f} per unit), samples {ts:.0f}")
    agg = collections.OrderedDict()
    for x in d:
        k = (x["addr"] - base) // region
        a = agg.setdefault(k, [0.0, 0.0])
        a[0] += x["inst"]
        a[1] += x["samp"]
    for k, (i, s) in agg.items():
        if i > 0.003 * ti or s > 0.003 * ts:
            print(f"  {hex(k * region):>8}  {100 * i / ti:5.1f}% inst  {100 * s / ts:5.1f}% samp")
    print("top instructions by stall samples:")
    for x in sorted(d, key=lambda x: -x["samp"])[:top]:
        rs = sorted(((x[k], k[6:]) for k in REASONS), reverse=True)[:3]
        why = " ".join(f"{n}={v / max(x['samp'], 1):.2f}" for v, n in rs if v > 0)
        print(f"  {100 * x['samp'] / ts:5.2f}%  {hex(x['addr'] - base):>7}  {x['inst']:10.0f}  {x['src'][:58]:58s} {why}")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], int(a[1], 0) if len(a) > 1 else 0x400, float(a[2]) if len(a) > 2 else 1,
         int(a[3]) if len(a) > 3 else 25)
