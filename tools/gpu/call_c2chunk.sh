for w in C2 C3; do
for cm in 0 1000 600 20000; do
  for pre in 0 1; do
  env FOFSE_CHUNK_MIN=$cm FOFSE_PRE_STREAM=$pre timeout 600 python bench.py --workload $w --no-cpu-baseline --no-parity --no-fp64 --steps 5 --warmup 3 > gpurun_out/c2c.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/c2c.json').read().strip().splitlines()[-1]); print('$w chunk_min=$cm pre=$pre', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['detail']['guard_reruns_per_step'])"
  done
done; done
