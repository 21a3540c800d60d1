set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s3m_build.log 2>&1; echo build rc=$?
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/s3m_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s3m_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3m_smoke.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/s3m_smoke.log
timeout 900 python bench.py > gpurun_out/s3m_bench.json 2> gpurun_out/s3m_bench.err; echo bench rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/s3m_bench.json').read().strip().splitlines()[-1]); print('C4', round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['roofline']['k1']['frac'], d['parity']['blocks_over_0.5'], d['parity']['max_px'], d['clocks'], d['gpu_launches'], d['detail']['fp64']['value'], d['detail']['fp64']['e2e']['value'], d['cpu_baseline']['value'])"
timeout 900 python bench.py --impl reference > gpurun_out/s3m_ref.json 2>/dev/null; echo ref rc=$?
for w in C1 C2 C3 C5; do
timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/s3m_$w.json 2>/dev/null; echo $w rc=$?
done
