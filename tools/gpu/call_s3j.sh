timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s3j_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/s3j_tests.log
timeout 900 python tools/parity_study_batch.py C3 4 300 4:1e-5 2>&1 | grep C3
bash tools/gpu/abn.sh s3j 2 FOFSE_HEAD_TIE=0 FOFSE_HEAD_TIE=1
WORKLOAD=C3 bash tools/gpu/abn.sh s3j3 2 FOFSE_HEAD_TIE=0 FOFSE_HEAD_TIE=1
WORKLOAD=C2 bash tools/gpu/abn.sh s3j2 1 FOFSE_HEAD_TIE=0 FOFSE_HEAD_TIE=1
WORKLOAD=C5 bash tools/gpu/abn.sh s3j5 1 FOFSE_HEAD_TIE=0 FOFSE_HEAD_TIE=1
