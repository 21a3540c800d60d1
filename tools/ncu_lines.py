"""Per-source-line hot spots of an ncu report (needs -lineinfo + --import-source).

Uses the combined CUDA+SASS source view (one row per SASS instruction with its
CUDA line) and aggregates stall samples and executed instructions per line."""
import csv, io, subprocess, sys
from collections import defaultdict


def main(path, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    agg = defaultdict(lambda: [0.0, 0.0, ""])
    fname, hdr = "", None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) < len(hdr):
            continue
        try:
            samp = float(r[4] or 0)
            inst = float(r[7] or 0)
        except ValueError:
            continue
        a = agg[(fname, r[0])]
        a[0] += samp
        a[1] += inst
        if r[1].strip():
            a[2] = r[1].strip()[:90]
    res = sorted(((v[0], v[1], k[0], k[1], v[2]) for k, v in agg.items()), reverse=True)
    tot = sum(x[0] for x in res) or 1
    toti = sum(x[1] for x in res) or 1
    print(f"total samples {tot:.0f}, instructions {toti:.3e}")
    for s, i, f, ln, src in res[:top]:
        print(f"{100*s/tot:5.1f}% samp {100*i/toti:5.1f}% inst  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
