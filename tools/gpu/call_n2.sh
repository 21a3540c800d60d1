FOFSE_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --parity-frames 8 > gpurun_out/bench_n2_gloo.json 2> gpurun_out/bench_n2_gloo.err; echo "n2 rc=$?"
tail -1 gpurun_out/bench_n2_gloo.json | cut -c1-600
timeout 600 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > /dev/null 2>&1; echo ref rc=$?
