set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/hx_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/hx_tests.log
timeout 600 python bench.py --workload C5 --no-cpu-baseline --no-fp64 --steps 5 --warmup 3 > gpurun_out/hx_c5.json 2>gpurun_out/hx_c5.err; echo c5 rc=$?
tail -2 gpurun_out/hx_c5.err
python -c "
import json; d=json.loads(open('gpurun_out/hx_c5.json').read().strip().splitlines()[-1]); print('C5', round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['parity'])"
WORKLOAD=C5 bash tools/gpu/abn.sh hx 2 FOFSE_ETR=0 FOFSE_ETR=1
