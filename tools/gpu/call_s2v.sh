set -x
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k2v2x_kernel --launch-skip 2 -c 1 -o gpurun_out/s2v_prof_k2v2x python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/s2v_ncu.log 2>&1; echo ncu rc=$?
