set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_C4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/r02_launches_C4.log 2>&1; echo ncu1 rc=$?
python tools/launch_summary.py gpurun_out/r02_launches_C4.csv 2>&1 | head -16
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k2v2r_kernel --launch-skip 2 -c 1 -o gpurun_out/r02_prof_k2v2r python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/r02_ncu_k2v2r.log 2>&1; echo ncu2 rc=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k1f_kernel --launch-skip 2 -c 1 -o gpurun_out/r02_prof_k1f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/r02_ncu_k1f.log 2>&1; echo ncu3 rc=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k2dcx_kernel --launch-skip 1 -c 1 -o gpurun_out/r02_prof_k2dcx python bench.py --workload C5 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/r02_ncu_k2dcx.log 2>&1; echo ncu4 rc=$?
ls -la gpurun_out/*.ncu-rep
