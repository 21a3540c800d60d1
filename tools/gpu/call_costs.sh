# what the guard re-runs and the fp64 head cost inside the overlapped C4 step
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
for opt in "" "--guard-tau 0" "--fp64-head 0" "--fp64-head 0 --guard-tau 0" ""; do
  timeout 600 python bench.py --no-cpu-baseline --no-parity --no-fp64 --steps 5 --warmup 3 $opt > gpurun_out/cost.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/cost.json').read().strip().splitlines()[-1])
print('opt=[$opt]', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],2), d['detail']['guard_reruns_per_step'], round(d['detail']['k1_ms'],2))"
done
