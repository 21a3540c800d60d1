set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -n 5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo "bench rc=$?"
FOFSE_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --frames 16 --no-cpu-baseline --parity-frames 4 > gpurun_out/bench_n2_gloo.json 2> gpurun_out/bench_n2_gloo.err; echo "n2 rc=$?"
timeout 600 python tools/parity_study.py C5 10 900 -1:-1 > gpurun_out/ps2_c5.log 2>&1
timeout 600 python tools/parity_study.py C3 4 310 -1:-1 > gpurun_out/ps2_c3.log 2>&1
timeout 600 python tools/parity_study.py C2 32 710 -1:-1 > gpurun_out/ps2_c2.log 2>&1
tail -n 3 gpurun_out/ps2_*.log
