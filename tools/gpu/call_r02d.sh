set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -n 15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-parity > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_r02d.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["detail"]["real_iterate_ms"], d["detail"]["k1_ms"], d["detail"].get("fp64",{}).get("value"))
PY
