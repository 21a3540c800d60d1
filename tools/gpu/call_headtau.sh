for s in 2207 9100; do timeout 900 python tools/parity_study_batch.py C4 256 $s 8:1e-5 6:1e-5 6:2e-5 4:2e-5 4:4e-5; done
for opt in "--fp64-head 8 --guard-tau 1e-5" "--fp64-head 6 --guard-tau 2e-5" "--fp64-head 4 --guard-tau 2e-5" "--fp64-head 4 --guard-tau 4e-5" "--fp64-head 6 --guard-tau 1e-5"; do
  timeout 600 python bench.py --no-cpu-baseline --no-parity --no-fp64 --steps 5 --warmup 3 $opt > gpurun_out/ht.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ht.json').read().strip().splitlines()[-1]); print('bench [$opt]', round(d['value']), round(d['e2e']['value']), d['detail']['guard_reruns_per_step'])"
done
