timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s3o_t.log 2>&1; echo t rc=$?; tail -1 gpurun_out/s3o_t.log
WORKLOAD=C3 bash tools/gpu/abn.sh s3o3 2 FOFSE_HEAD_TIE=0 FOFSE_AB=new
bash tools/gpu/abn.sh s3o 2 FOFSE_HEAD_TIE=0 FOFSE_AB=new
WORKLOAD=C5 bash tools/gpu/abn.sh s3o5 1 FOFSE_HEAD_TIE=0 FOFSE_AB=new
