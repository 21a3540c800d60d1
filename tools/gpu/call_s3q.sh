FOFSE_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --parity-frames 8 > gpurun_out/s3q_n2.json 2> gpurun_out/s3q_n2.err; echo n2 rc=$?
tail -1 gpurun_out/s3q_n2.json | cut -c1-250
python -c "
import json; d=json.loads(open('gpurun_out/s3q_n2.json').read().strip().splitlines()[-1]); print(d.get('parity',{}).get('blocks_over_0.5'), d.get('parallelism'))"
