set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_C4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/r02_launches_C4.log 2>&1; echo ncu1 rc=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k2v2r_kernel --launch-skip 2 -c 1 -o gpurun_out/r02_prof_k2v2r python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/r02_ncu_k2v2r.log 2>&1; echo ncu2 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_C5.csv python bench.py --workload C5 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu3 rc=$?
for w in C1 C2 C4; do timeout 600 python bench.py --workload $w --precision fp64 --no-cpu-baseline --no-parity --steps 5 --warmup 3 > gpurun_out/f64b_$w.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/f64b_$w.json').read().strip().splitlines()[-1]); print('$w fp64', round(d['value']), round(d['e2e']['value']), d['ms_per_step'])"; done
