set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "T128 or C5 or C2 or fp32 or border" > gpurun_out/hq_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/hq_tests.log
WORKLOAD=C5 bash tools/gpu/abn.sh hq5 3 FOFSE_V2H_QK=0 FOFSE_V2H_QK=1
WORKLOAD=C2 bash tools/gpu/abn.sh hq2 3 FOFSE_V2H_QK=0 FOFSE_V2H_QK=1
timeout 600 python bench.py --workload C5 --no-cpu-baseline --no-fp64 --steps 5 --warmup 3 > gpurun_out/hq_c5.json 2>/dev/null; echo c5 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/hq_c5.json').read().strip().splitlines()[-1]); print('C5', round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['parity']['blocks_over_0.5'], d['parity']['guard_reruns'], d['parity']['max_px'])"
