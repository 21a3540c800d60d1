set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'k2d_kernel<\(int\)64, \(bool\)0, \(bool\)0, \(bool\)0, \(bool\)0>' --launch-skip 3 -c 1 -o gpurun_out/r02_prof_head python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/r02_ncu_head.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'k2d_kernel<\(int\)64, \(bool\)0, \(bool\)1, \(bool\)0, \(bool\)0>' --launch-skip 2 -c 1 -o gpurun_out/r02_prof_replay python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/r02_ncu_replay.log 2>&1; echo ncu2 rc=$?
