# A/B of diagnostic variants on ONE box: bench.py C4 (value only) alternating env settings
# usage: bash tools/gpu/ab.sh NAME "ENV_A" "ENV_B" [reps]
name=$1; A=$2; B=$3; reps=${4:-3}
for r in $(seq $reps); do
  for v in A B; do
    if [ $v = A ]; then E=$A; else E=$B; fi
    env $E timeout 600 python bench.py --workload ${WORKLOAD:-C4} --no-cpu-baseline --no-parity --no-fp64 --steps 5 --warmup 3 > gpurun_out/ab_${name}_${v}_$r.json 2>/dev/null
    python -c "
import json,sys
d=json.loads(open('gpurun_out/ab_${name}_${v}_$r.json').read().strip().splitlines()[-1])
print('$v', '$E', round(d['value']), round(d['e2e']['value']), round(d['roofline']['frac'],4), round(d['detail']['real_iterate_ms'],2))"
  done
done
