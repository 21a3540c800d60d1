set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/k1h_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/k1h_tests.log
timeout 900 python bench.py --no-cpu-baseline --no-fp64 --steps 5 --warmup 3 > gpurun_out/k1h_c4.json 2>gpurun_out/k1h_c4.err; echo c4 rc=$?
tail -3 gpurun_out/k1h_c4.err
python -c "
import json; d=json.loads(open('gpurun_out/k1h_c4.json').read().strip().splitlines()[-1]); print('C4', round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['parity'])"
bash tools/gpu/abn.sh k1h 2 FOFSE_K1H=0 FOFSE_K1H=1
