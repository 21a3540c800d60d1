set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
timeout 900 python -m pytest tests -m gpu -x -q -k "frame or fp64 or exact" > gpurun_out/f64pipe_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/f64pipe_tests.log
for w in C4 C2 C1; do timeout 600 python bench.py --workload $w --precision fp64 --no-cpu-baseline --no-parity --steps 5 --warmup 3 > gpurun_out/f64p_$w.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/f64p_$w.json').read().strip().splitlines()[-1]); print('$w fp64', round(d['value']), round(d['e2e']['value']), d['ms_per_step'])"; done
