set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size
timeout 900 ncu --metrics $M --clock-control none -k regex:k2v2h_kernel --launch-skip 1 -c 1 --csv python bench.py --workload C5 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/r02_dram_C5.csv 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:k2v2r_kernel --launch-skip 1 -c 1 --csv python bench.py --workload C3 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/r02_dram_C3.csv 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:k2v2 --launch-skip 2 -c 1 --csv python bench.py --workload C2 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > gpurun_out/r02_dram_C2.csv 2>&1
FOFSE_HOST_PROF=1 timeout 300 python bench.py --workload C2 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2> gpurun_out/r02_hostprof_C2.err
FOFSE_HOST_PROF=1 timeout 300 python bench.py --workload C3 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2> gpurun_out/r02_hostprof_C3.err
FOFSE_HOST_PROF=1 timeout 300 python bench.py --workload C5 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2> gpurun_out/r02_hostprof_C5.err
for w in C2 C3 C5; do grep -h "k2v2" gpurun_out/r02_dram_$w.csv | head -8; done
