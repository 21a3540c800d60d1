set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "T128 or C5 or t128" > gpurun_out/pytest_t128.log 2>&1; echo "t128 rc=$?"
tail -n 30 gpurun_out/pytest_t128.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -n 8 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --workload C5 --no-cpu-baseline --no-parity --steps 5 --warmup 3 > gpurun_out/r02f_C5.json 2> gpurun_out/r02f_C5.err
timeout 600 python bench.py --workload C2 --precision fp64 --no-cpu-baseline --no-parity --steps 5 --warmup 3 > gpurun_out/r02f_C2f64.json 2> gpurun_out/r02f_C2f64.err
python - <<'PY'
import json
for w in ["C5","C2f64"]:
    try:
        d=json.loads(open(f"gpurun_out/r02f_{w}.json").read().strip().splitlines()[-1])
        print(w, round(d["value"]), round(d["e2e"]["value"]), d["roofline"]["frac"], d["ms_per_step"], d["detail"]["guard_reruns_per_step"], d["detail"].get("fp64",{}).get("value"))
    except Exception as e: print(w, "ERR", e)
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches_C5.csv python bench.py --workload C5 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu rc=$?
python tools/launch_summary.py gpurun_out/r02f_launches_C5.csv 2>&1 | head -14
