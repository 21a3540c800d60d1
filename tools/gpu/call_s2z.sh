set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2z_launches_C4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu1 rc=$?
python tools/launch_summary.py gpurun_out/s2z_launches_C4.csv 2>&1 | head -18
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2z_launches_C5.csv python bench.py --workload C5 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu2 rc=$?
python tools/launch_summary.py gpurun_out/s2z_launches_C5.csv 2>&1 | head -14
