"""Aggregate an ncu SASS source page by opcode: stall samples + instructions."""
import csv, io, re, subprocess, sys
from collections import defaultdict

def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    agg = defaultdict(lambda: [0.0, 0.0, 0])
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        src = d["Source"].strip()
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", src)
        op = m.group(2) if m else src[:10]
        try:
            agg[op][0] += float(d["Warp Stall Sampling (All Samples)"] or 0)
            agg[op][1] += float(d["Instructions Executed"] or 0)
            agg[op][2] += 1
        except ValueError:
            pass
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    for op, (s, i, n) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"{op:10s} inst {100*i/ti:5.1f}%  stall-samples {100*s/ts:5.1f}%  ({n} sites)")

if __name__ == "__main__":
    main(sys.argv[1])
