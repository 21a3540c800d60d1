set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s2u_build.log 2>&1; echo build rc=$?
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/s2u_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s2u_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2u_smoke.log 2>&1; echo smoke rc=$?
tail -1 gpurun_out/s2u_smoke.log
timeout 900 python bench.py > gpurun_out/s2u_bench.json 2> gpurun_out/s2u_bench.err; echo bench rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/s2u_bench.json').read().strip().splitlines()[-1]); print('C4', round(d['value']), round(d['e2e']['value']), d['roofline']['frac'], d['roofline']['k1']['frac'], d['parity']['blocks_over_0.5'], d['parity']['max_px'], d['clocks'], d['gpu_launches'], d['detail']['fp64']['value'], d['detail']['fp64']['e2e']['value'], d['cpu_baseline']['value'])"
timeout 900 python bench.py --impl reference > gpurun_out/s2u_ref.json 2>/dev/null; echo ref rc=$?
FOFSE_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --parity-frames 8 > gpurun_out/s2u_n2.json 2> gpurun_out/s2u_n2.err; echo n2 rc=$?
tail -1 gpurun_out/s2u_n2.json | cut -c1-300
