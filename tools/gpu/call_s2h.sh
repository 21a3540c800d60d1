set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1p_kernel --launch-skip 3 -c 1 -o gpurun_out/s2h_prof_k1p python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/s2h_ncu_k1p.log 2>&1; echo ncu rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2h_launches_C4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu2 rc=$?
python tools/launch_summary.py gpurun_out/s2h_launches_C4.csv 2>&1 | head -16
