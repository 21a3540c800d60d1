set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/etr_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/etr_tests.log
timeout 900 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/etr_c4.json 2>gpurun_out/etr_c4.err; echo c4 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/etr_c4.json').read().strip().splitlines()[-1]); print('C4', round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['parity'], d['detail']['fp64'])"
FOFSE_ETR=0 timeout 900 python bench.py --no-cpu-baseline --no-fp64 --steps 3 --warmup 3 > gpurun_out/etr0_c4.json 2>/dev/null; echo replay rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/etr0_c4.json').read().strip().splitlines()[-1]); print('REPLAY', round(d['value']), d['parity'])"
