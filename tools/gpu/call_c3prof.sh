set -x
timeout 600 python bench.py --workload C3 --no-cpu-baseline --no-parity --no-fp64 --steps 5 --warmup 3 > gpurun_out/c3_bench.json 2>/dev/null; echo bench rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_C3.csv python bench.py --workload C3 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k2v2r_kernel --launch-skip 1 -c 1 -o gpurun_out/r02_prof_k2v2r32 python bench.py --workload C3 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu2 rc=$?
