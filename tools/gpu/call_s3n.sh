FOFSE_HOST_PROF=1 timeout 600 python bench.py --workload C3 --no-cpu-baseline --no-parity --no-fp64 --steps 1 --warmup 3 > /dev/null 2> gpurun_out/s3n_c3.err; echo rc=$?
tail -16 gpurun_out/s3n_c3.err
