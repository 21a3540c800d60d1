set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
timeout 600 python -m pytest tests/test_gpu_exact.py -x -q > gpurun_out/pytest_exact.log 2>&1; echo "exact rc=$?"
tail -n 30 gpurun_out/pytest_exact.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -n 15 gpurun_out/pytest_gpu.log
for w in C1 C2; do timeout 300 python bench.py --workload $w --precision fp64 --steps 5 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/b64_$w.json 2> gpurun_out/b64_$w.err; done
timeout 300 python bench.py --workload C2 --steps 5 --warmup 3 --no-cpu-baseline --no-fp64 > gpurun_out/b32_C2.json 2> gpurun_out/b32_C2.err
python - <<'PY'
import json
for f in ["b64_C1","b64_C2","b32_C2"]:
    try:
        d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1]); print(f, d["value"], d["e2e"]["value"], d["detail"]["guard_reruns_per_step"], d["roofline"]["frac"])
    except Exception as e: print(f, "ERR", e)
PY
