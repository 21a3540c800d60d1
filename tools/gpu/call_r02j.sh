set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
timeout 900 python tools/parity_study.py C3 6 321 -1:-1 > gpurun_out/ps3_c3.log 2>&1; cat gpurun_out/ps3_c3.log
timeout 900 python tools/parity_study.py C3 4 777 -1:-1 >> gpurun_out/ps3_c3.log 2>&1; tail -2 gpurun_out/ps3_c3.log
WORKLOAD=C3 bash tools/gpu/ab.sh head32 "FOFSE_DUMMY=0" "FOFSE_DUMMY=1" 1
timeout 600 python bench.py --workload C3 --fp64-head 8 --no-cpu-baseline --no-parity --no-fp64 --steps 5 --warmup 3 > gpurun_out/c3_h8.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/c3_h8.json').read().strip().splitlines()[-1]); print('head8', round(d['value']), round(d['e2e']['value']), d['roofline']['frac'])"
