for w in C5 C4; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-fp64 --steps 5 --warmup 3 > gpurun_out/c5c2.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/c5c2.json').read().strip().splitlines()[-1]); print('$w', round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['roofline']['frac'], d['parity']['blocks_over_0.5'], d['parity']['max_px'])"
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
