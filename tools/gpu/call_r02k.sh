set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 4 gpurun_out/pytest_gpu.log
for w in C4 C5 C2 C3; do timeout 600 python bench.py --workload $w --no-cpu-baseline --no-parity --no-fp64 --steps 5 --warmup 3 > gpurun_out/r02k_$w.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r02k_$w.json').read().strip().splitlines()[-1]); print('$w', round(d['value']), round(d['e2e']['value']), round(d['roofline']['frac'],4), d['ms_per_step'], d['detail']['guard_reruns_per_step'])"; done
timeout 600 python tools/parity_study.py C5 8 620 -1:-1 | tail -2
timeout 600 python tools/parity_study.py C2 32 720 -1:-1 | tail -2
