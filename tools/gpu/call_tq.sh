set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "small_transforms or C3 or edge or determinism" > gpurun_out/tq_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/tq_tests.log
WORKLOAD=C3 bash tools/gpu/abn.sh tq 3 FOFSE_V2T_QK=0 FOFSE_V2T_QK=1
timeout 600 python bench.py --workload C3 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/tq_c3.json 2>/dev/null; echo c3 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/tq_c3.json').read().strip().splitlines()[-1]); print('C3', round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['parity']['blocks_over_0.5'], d['parity']['guard_reruns'], d['parity']['max_px'])"
