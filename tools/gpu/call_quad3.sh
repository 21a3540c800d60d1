set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/quad3_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/quad3_tests.log
bash tools/gpu/abn.sh q3 2 FOFSE_V2R_VAR=1 FOFSE_V2R_VAR=0
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/q3_c4.json 2>gpurun_out/q3_c4.err; echo c4 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/q3_c4.json').read().strip().splitlines()[-1]); print('C4', round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['parity']['blocks_over_0.5'], d['parity']['guard_reruns'], d['detail']['fp64'])"
