B=$PWD/paper_2207_01205_b200/_lib/libfofse_base.so
for w in C1 C5; do for r in 1 2; do for v in "FOFSE_LIB_PATH=$B" "FOFSE_AB=new"; do
  prec=fp32; [ $w = C1 ] && prec=fp64
  env $v timeout 600 python bench.py --workload $w --precision $prec --no-cpu-baseline --no-parity --no-fp64 --steps 5 --warmup 3 > gpurun_out/nd3.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/nd3.json').read().strip().splitlines()[-1]); print('$w', '$v'[:20], round(d['value']), round(d['e2e']['value']), d['ms_per_step'])"
done; done; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
