set -x
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k2v2c_kernel --launch-skip 1 -c 1 -o gpurun_out/s3a_prof_k2v2c python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/s3a_ncu.log 2>&1; echo ncu rc=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:'k2d_kernel' --launch-skip 3 -c 1 -o gpurun_out/s3a_prof_head python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/s3a_ncu2.log 2>&1; echo ncu2 rc=$?
