for opt in "" "--guard-tau 0"; do
  timeout 600 python bench.py --workload C5 --no-cpu-baseline --no-parity --no-fp64 --steps 5 --warmup 3 $opt > gpurun_out/c5cost.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/c5cost.json').read().strip().splitlines()[-1])
print('opt=[$opt]', round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],2), d['detail']['guard_reruns_per_step'], d['detail'].get('real_iterate_ms'))"
done
timeout 300 env FOFSE_HOST_PROF=1 python bench.py --workload C5 --no-cpu-baseline --no-parity --no-fp64 --steps 1 --warmup 3 > /dev/null 2> gpurun_out/c5tl.err
grep "fofse chunk\|fofse guard" gpurun_out/c5tl.err | tail -8
