set -x
B=$PWD/paper_2207_01205_b200/_lib/libfofse_base.so
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s2r_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s2r_tests.log
bash tools/gpu/abn.sh s2r 3 FOFSE_LIB_PATH=$B FOFSE_AB=new
WORKLOAD=C5 bash tools/gpu/abn.sh s2r5 2 FOFSE_LIB_PATH=$B FOFSE_AB=new
WORKLOAD=C2 bash tools/gpu/abn.sh s2r2 2 FOFSE_LIB_PATH=$B FOFSE_AB=new
