"""K3 (the synthesis fused into an iteration kernel's epilogue) as a share of
that kernel: instructions executed and warp-stall samples attributed to the
source lines of v2_finish (csrc/v2common.cuh) in an ncu report captured with
--import-source on and -lineinfo.

usage: python tools/ncu_k3_share.py REPORT
"""
import csv
import io
import re
import subprocess
import sys

V2 = "paper_2207_01205_b200/csrc/v2common.cuh"


def finish_range(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if re.search(r"void v2_finish\(", l)) - 1  # the template line
    return start + 1, len(lines)  # 1-based, to the end of the file (v2_finish is its last function)


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    lo, hi = finish_range(V2)
    tot_i = tot_s = k3_i = k3_s = 0.0
    cur = None
    hdr = None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            cur = row[1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or not row[0].isdigit():
            continue
        try:
            inst = float(row[hdr.index("Instructions Executed")] or 0)
            samp = float(row[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        tot_i += inst
        tot_s += samp
        if cur and cur.endswith("v2common.cuh") and lo <= int(row[0]) <= hi:
            k3_i += inst
            k3_s += samp
    print(f"report {rep}")
    print(f"v2_finish (fused synthesis + write-back, {V2}:{lo}-{hi})")
    print(f"  instructions executed: {k3_i:.4g} of {tot_i:.4g} = {100 * k3_i / max(tot_i, 1):.1f} %")
    print(f"  warp-stall samples:    {k3_s:.4g} of {tot_s:.4g} = {100 * k3_s / max(tot_s, 1):.1f} %")


if __name__ == "__main__":
    main(sys.argv[1])
