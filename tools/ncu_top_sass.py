"""Top SASS instructions by warp-stall samples (ncu source page, SASS view)."""
import csv, io, subprocess, sys

def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    recs = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        try:
            s = float(d["Warp Stall Sampling (All Samples)"] or 0)
        except ValueError:
            continue
        recs.append((s, d["Address"], d["Source"].strip()[:80], d.get("Warp Stall Sampling (Not-issued Samples)", "")))
    tot = sum(x[0] for x in recs) or 1
    print(f"total samples {tot:.0f}")
    for s, a, src, ni in sorted(recs, reverse=True)[:top]:
        print(f"{100*s/tot:5.2f}%  {a}  {src}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
