set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f3_build.log 2>&1; echo build rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/f3_tests.log 2>&1; echo tests rc=$?
tail -1 gpurun_out/f3_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/f3_smoke.log
timeout 900 python bench.py > gpurun_out/f3_bench.json 2> gpurun_out/f3_bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/f3_ref.json 2>/dev/null; echo ref rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/f3_bench.json').read().strip().splitlines()[-1]); print('C4', round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['parity']['blocks_over_0.5'], d['parity']['max_px'], d['clocks'], d['gpu_launches'], d['detail']['fp64']['value'])
r=json.loads(open('gpurun_out/f3_ref.json').read().strip().splitlines()[-1]); print('REF', r['value'], r.get('impl'))"
