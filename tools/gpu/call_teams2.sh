set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "small_transforms or C3 or edge or determinism" > gpurun_out/teams_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/teams_tests.log
B=$PWD/paper_2207_01205_b200/_lib/libfofse_base.so; N=$PWD/paper_2207_01205_b200/_lib/libfofse.so
timeout 600 python tools/lib_ab_outputs.py C3 1 $B $N
WORKLOAD=C3 bash tools/gpu/ab.sh teams2 "FOFSE_LIB_PATH=$B" "FOFSE_AB=new" 2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k2v2t_kernel --launch-skip 1 -c 1 -o gpurun_out/r02_prof_k2v2t32b python bench.py --workload C3 --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu rc=$?
