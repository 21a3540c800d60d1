timeout 300 env FOFSE_HOST_PROF=1 python bench.py --workload C3 --no-cpu-baseline --no-parity --no-fp64 --steps 2 --warmup 3 > gpurun_out/c3host.json 2> gpurun_out/c3host.err; echo rc=$?
grep "fofse host" gpurun_out/c3host.err | tail -40
