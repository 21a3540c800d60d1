timeout 300 env FOFSE_HOST_PROF=1 python bench.py --no-cpu-baseline --no-parity --no-fp64 --steps 1 --warmup 3 > gpurun_out/tl.json 2> gpurun_out/tl.err; echo rc=$?
