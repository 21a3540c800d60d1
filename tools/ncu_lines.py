"""Per-source-line hot spots of an ncu report (needs -lineinfo + --import-source)."""
import csv, io, subprocess, sys

def main(path, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    res = []
    fname = ""
    for r in rows:
        if r and r[0] == "File Name":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        try:
            samp = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            inst = float(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        if samp or inst:
            res.append((samp, inst, fname, d["Line No"], d["Source"].strip()[:90]))
    tot = sum(x[0] for x in res) or 1
    toti = sum(x[1] for x in res) or 1
    res.sort(reverse=True)
    print(f"total samples {tot:.0f}, instructions {toti:.3e}")
    for s, i, f, ln, src in res[:top]:
        print(f"{100*s/tot:5.1f}% samp {100*i/toti:5.1f}% inst  {f}:{ln}  {src}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
