# round-robin A/B/C... of env settings on ONE box: bench.py (WORKLOAD, default C4), value only
# usage: bash tools/gpu/abn.sh NAME REPS "ENV1" "ENV2" ...
name=$1; reps=$2; shift 2
for r in $(seq $reps); do
  i=0
  for E in "$@"; do
    i=$((i+1))
    env $E timeout 600 python bench.py --workload ${WORKLOAD:-C4} --no-cpu-baseline --no-parity --no-fp64 --steps 5 --warmup 3 > gpurun_out/abn_${name}_${i}_$r.json 2>/dev/null
    python -c "
import json
d=json.loads(open('gpurun_out/abn_${name}_${i}_$r.json').read().strip().splitlines()[-1])
print('$i', '$E', round(d['value']), round(d['e2e']['value']), round(d['roofline']['frac'],4), round(d['detail']['real_iterate_ms'],2), round(d['detail'].get('k1_ms',0),2), round(d['detail'].get('init_ms',0),2))"
  done
done
