set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s2a_build.log 2>&1; echo build rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s2a_tests.log 2>&1; echo tests rc=$?
tail -1 gpurun_out/s2a_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2a_smoke.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/s2a_smoke.log
timeout 900 python bench.py > gpurun_out/s2a_bench.json 2> gpurun_out/s2a_bench.err; echo bench rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/s2a_bench.json').read().strip().splitlines()[-1]); print('C4', round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['parity']['blocks_over_0.5'], d['parity']['max_px'], d['clocks'], d['gpu_launches'], d['detail']['fp64']['value'])"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'k2d_kernel<\(int\)64, \(bool\)0, \(bool\)0, \(bool\)0, \(bool\)0, \(bool\)0>' --launch-skip 3 -c 1 -o gpurun_out/s2a_prof_head python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/s2a_ncu_head.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1f_kernel --launch-skip 3 -c 1 -o gpurun_out/s2a_prof_k1f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/s2a_ncu_k1f.log 2>&1; echo ncu2 rc=$?
ls -la gpurun_out/*.ncu-rep
