B=/root/repo/paper_2207_01205_b200/_lib/libfofse_base.so
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for r in 1 2; do for v in "FOFSE_LIB_PATH=$B" "FOFSE_AB=new"; do
  env $v timeout 600 python bench.py --precision fp64 --no-cpu-baseline --no-parity --no-fp64 --steps 3 --warmup 2 > gpurun_out/tw64.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/tw64.json').read().strip().splitlines()[-1]); print('fp64', '$v'[:20], round(d['value']), round(d['e2e']['value']), d['ms_per_step'])"
done; done
WORKLOAD=C5 bash tools/gpu/abn.sh tw5 2 FOFSE_LIB_PATH=$B FOFSE_AB=new
bash tools/gpu/abn.sh tw4 1 FOFSE_LIB_PATH=$B FOFSE_AB=new
