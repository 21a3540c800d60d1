set -x
for w in C5 C2 C3; do
timeout 600 python bench.py --workload $w --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/s2c_$w.json 2>/dev/null; echo $w rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/s2c_$w.json').read().strip().splitlines()[-1]); print('$w', round(d['value']), round(d['e2e']['value']), round(d['roofline']['frac'],4), d.get('parity',{}).get('blocks_over_0.5'), d['detail'].get('guard_reruns_per_step'))"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2c_launches_C5.csv python bench.py --workload C5 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu1 rc=$?
python tools/launch_summary.py gpurun_out/s2c_launches_C5.csv 2>&1 | head -16
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2c_launches_C4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu2 rc=$?
python tools/launch_summary.py gpurun_out/s2c_launches_C4.csv 2>&1 | head -16
