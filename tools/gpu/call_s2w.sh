set -x
B=$PWD/paper_2207_01205_b200/_lib/libfofse_base.so
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s2w_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s2w_tests.log
bash tools/gpu/abn.sh s2w 3 FOFSE_LIB_PATH=$B FOFSE_AB=new
