set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/s3p_tests.log 2>&1; echo tests rc=$?
tail -1 gpurun_out/s3p_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3p_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/s3p_bench.json 2> gpurun_out/s3p_bench.err; echo bench rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/s3p_bench.json').read().strip().splitlines()[-1]); print('C4', round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['roofline']['k1']['frac'], d['parity']['blocks_over_0.5'], d['parity']['max_px'], d['clocks'], d['gpu_launches'], d['detail']['fp64']['value'], d['detail']['fp64']['e2e']['value'], d['cpu_baseline']['value'])"
for w in C2 C3 C5; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/s3p_$w.json 2>/dev/null; echo $w rc=$?; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3p_launches_C4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu rc=$?
python tools/launch_summary.py gpurun_out/s3p_launches_C4.csv 2>&1 | head -18
