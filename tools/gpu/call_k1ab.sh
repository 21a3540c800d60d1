# K1f variant vs the base build (FOFSE_LIB_PATH), tests, ncu of the new K1f
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "init or spectra or conceal or frame" > gpurun_out/k1ab_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/k1ab_tests.log
bash tools/gpu/ab.sh k1 "FOFSE_LIB_PATH=$PWD/paper_2207_01205_b200/_lib/libfofse_base.so" "FOFSE_AB=new" 2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1f_kernel --launch-skip 6 -c 1 -o gpurun_out/r02_prof_k1f_b python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu rc=$?
