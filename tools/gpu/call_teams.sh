# K2v2t (several lost blocks per warp at T <= 32): tests, output identity vs the base build, C3/C4 benches
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/teams_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/teams_tests.log
B=$PWD/paper_2207_01205_b200/_lib/libfofse_base.so; N=$PWD/paper_2207_01205_b200/_lib/libfofse.so
timeout 600 python tools/lib_ab_outputs.py C3 1 $B $N
timeout 600 python tools/lib_ab_outputs.py C4 4 $B $N
WORKLOAD=C3 bash tools/gpu/ab.sh teams "FOFSE_LIB_PATH=$B" "FOFSE_AB=new" 2
timeout 600 python bench.py --workload C3 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/teams_c3.json 2>/dev/null; echo c3 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/teams_c3.json').read().strip().splitlines()[-1]); print('C3', round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['parity'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k2v2t_kernel --launch-skip 1 -c 1 -o gpurun_out/r02_prof_k2v2t32 python bench.py --workload C3 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu rc=$?
