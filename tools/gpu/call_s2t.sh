set -x
FOFSE_HOST_PROF=1 timeout 600 python bench.py --workload C3 --no-cpu-baseline --no-parity --no-fp64 --steps 2 --warmup 3 > gpurun_out/s2t_c3.json 2> gpurun_out/s2t_c3.err; echo rc=$?
tail -60 gpurun_out/s2t_c3.err
