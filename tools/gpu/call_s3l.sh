timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s3l_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/s3l_tests.log
timeout 1200 python tools/parity_study_batch.py C2 32 700 8:1e-5 2>&1 | grep C2
timeout 1200 python tools/parity_study_batch.py C4 64 2207 8:1e-5 2>&1 | grep C4
timeout 1200 python tools/parity_study_batch.py C3 4 300 4:1e-5 2>&1 | grep C3
bash tools/gpu/abn.sh s3l 2 FOFSE_AB=new
WORKLOAD=C2 bash tools/gpu/abn.sh s3l2 1 FOFSE_AB=new
WORKLOAD=C3 bash tools/gpu/abn.sh s3l3 1 FOFSE_AB=new
