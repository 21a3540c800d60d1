"""Per-SASS-address execution counts of an ncu report grouped into classes (every
selection / non-self / self / per block): where a kernel's instructions go per unit.
usage: python tools/ncu_exec_classes.py REPORT [COUNT_TO_LIST]"""
import csv, io, subprocess, sys, collections
rep=sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
recs=[]
for r in rows[2:]:
    if len(r) < len(hdr): continue
    d = dict(zip(hdr, r))
    try:
        ex = float(d.get("Instructions Executed") or 0); samp=float(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError: continue
    recs.append((int(d["Address"],16) if d["Address"].startswith("0x") else 0, d["Source"].strip(), ex, samp))
recs.sort()
base=recs[0][0]
tot=sum(r[2] for r in recs)
# iteration count = max exec of a frequent instruction
freq=collections.Counter(round(r[2]) for r in recs if r[2]>0)
print("total warp inst", tot)
print("top exec counts", freq.most_common(8))
cls=collections.defaultdict(lambda:[0,0.0,0.0])
# per-unit normaliser: the largest execution count shared by many instructions (every selection)
NSEL=max((k for k, n in freq.items() if n >= 50), default=1)
for a,src,ex,s in recs:
    k=round(ex)
    cls[k][0]+=1; cls[k][1]+=ex; cls[k][2]+=s
print("exec-count classes by total instructions:")
for k,(n,e,s) in sorted(cls.items(), key=lambda kv:-kv[1][1])[:14]:
    print(f"  count {k:>10}  static {n:4d}  dyn share {100*e/tot:5.1f}%  per-iter {e/NSEL:6.1f}")
if len(sys.argv)>2:
    want=int(sys.argv[2])
    for a,src,ex,s in recs:
        if round(ex)==want: print(f"{a-base:05x} {src[:90]}")
