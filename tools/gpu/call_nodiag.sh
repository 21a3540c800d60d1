B=$PWD/paper_2207_01205_b200/_lib/libfofse_base.so
WORKLOAD=C3 bash tools/gpu/abn.sh nd3 2 FOFSE_LIB_PATH=$B FOFSE_AB=new
WORKLOAD=C5 bash tools/gpu/abn.sh nd5 2 FOFSE_LIB_PATH=$B FOFSE_AB=new
WORKLOAD=C2 bash tools/gpu/abn.sh nd2 2 FOFSE_LIB_PATH=$B FOFSE_AB=new
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
