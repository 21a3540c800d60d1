# exact near-tie resolution (K2v2x): parity + speed vs the fp64 REPLAY re-runs
set -x
timeout 900 python bench.py --no-cpu-baseline --no-fp64 --steps 3 --warmup 3 > gpurun_out/etr1.json 2>gpurun_out/etr1.err; echo etr rc=$?
tail -3 gpurun_out/etr1.err
python -c "
import json; d=json.loads(open('gpurun_out/etr1.json').read().strip().splitlines()[-1]); print('ETR', round(d['value']), round(d['e2e']['value']), d['parity'])"
FOFSE_ETR=0 timeout 900 python bench.py --no-cpu-baseline --no-fp64 --steps 3 --warmup 3 > gpurun_out/etr0.json 2>/dev/null; echo replay rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/etr0.json').read().strip().splitlines()[-1]); print('REPLAY', round(d['value']), round(d['e2e']['value']), d['parity'])"
