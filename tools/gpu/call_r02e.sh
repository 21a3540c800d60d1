set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
for w in C5 C3 C2 C1; do timeout 600 python bench.py --workload $w --no-cpu-baseline --no-parity --steps 5 --warmup 3 > gpurun_out/r02e_$w.json 2> gpurun_out/r02e_$w.err; done
python - <<'PY'
import json
for w in ["C5","C3","C2","C1"]:
    try:
        d=json.loads(open(f"gpurun_out/r02e_{w}.json").read().strip().splitlines()[-1])
        print(w, round(d["value"]), round(d["e2e"]["value"]), d["roofline"]["frac"], d["ms_per_step"], d["detail"]["guard_reruns_per_step"], d["detail"].get("fp64",{}).get("value"))
    except Exception as e: print(w, "ERR", e)
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_launches_C5.csv python bench.py --workload C5 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu rc=$?
python tools/launch_summary.py gpurun_out/r02e_launches_C5.csv 2>&1 | head -30
