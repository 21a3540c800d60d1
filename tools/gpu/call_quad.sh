# K2v2r quad keys (FOFSE_V2R_VAR=5): tests under the variant, same-box A/B, full C4 parity
set -x
FOFSE_V2R_VAR=5 timeout 1200 python -m pytest tests -m gpu -x -q -k "fp32 or C4 or frame or determinism or guard" > gpurun_out/quad_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/quad_tests.log
bash tools/gpu/ab.sh quad "FOFSE_V2R_VAR=0" "FOFSE_V2R_VAR=5" 3
FOFSE_V2R_VAR=5 timeout 900 python bench.py --no-cpu-baseline --no-fp64 --steps 5 --warmup 3 > gpurun_out/quad_c4.json 2>/dev/null; echo c4 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/quad_c4.json').read().strip().splitlines()[-1]); print('C4 quad', round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['parity'])"
