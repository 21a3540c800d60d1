"""Per-source-line instruction / stall-sample shares of an ncu report captured
with --import-source on (kernels compiled with -lineinfo).

usage: python tools/ncu_lines.py REPORT [TOP]
"""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, hdr, agg = None, None, {}
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        try:
            inst = float(r[hdr.index("Instructions Executed")] or 0)
            samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        k = (cur, int(r[0]))
        a = agg.setdefault(k, [0.0, 0.0, r[1].strip()[:80]])
        a[0] += inst
        a[1] += samp
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"report {rep}: {ti:.4g} warp instructions, {ts:.4g} stall samples")
    for (f, ln), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * i / ti:5.1f}% inst {100 * s / ts:5.1f}% samp  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
