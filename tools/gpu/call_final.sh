set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_final.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], "traffic", d["roofline"]["traffic"])
print("parity", d["parity"])
print("fp64", d["detail"]["fp64"])
print("cpu", d["cpu_baseline"])
print("k1", d["roofline"]["k1"]["frac"], "clocks", d["clocks"], "launches", d["gpu_launches"])
r=json.loads(open("gpurun_out/bench_ref.json").read().strip().splitlines()[-1])
print("ref", r["value"], r["cpu_baseline"]["sample"], r["config"]==d["config"])
PY
