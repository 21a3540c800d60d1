set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/twx_tests.log 2>&1; echo rc=$?; tail -1 gpurun_out/twx_tests.log
WORKLOAD=C3 bash tools/gpu/abn.sh twx3 2 FOFSE_LIB_PATH=$PWD/paper_2207_01205_b200/_lib/libfofse_base.so FOFSE_AB=new
bash tools/gpu/abn.sh twx4 1 FOFSE_LIB_PATH=$PWD/paper_2207_01205_b200/_lib/libfofse_base.so FOFSE_AB=new
