set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/etr_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/etr_tests.log
timeout 900 python bench.py --no-cpu-baseline --no-fp64 --steps 3 --warmup 3 > gpurun_out/etr1.json 2>gpurun_out/etr1.err; echo etr rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/etr1.json').read().strip().splitlines()[-1]); print('ETR', round(d['value']), round(d['e2e']['value']), d['parity'])"
bash tools/gpu/abn.sh etr 2 FOFSE_ETR=0 FOFSE_ETR=1
WORKLOAD=C2 bash tools/gpu/abn.sh etr2 2 FOFSE_ETR=0 FOFSE_ETR=1
