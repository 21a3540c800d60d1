timeout 900 python tools/parity_study_batch.py C3 4 300 4:1e-5 2>&1 | grep C3
timeout 900 python tools/parity_study_batch.py C3 4 900 4:1e-5 2>&1 | grep C3
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s3h_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/s3h_tests.log
bash tools/gpu/abn.sh s3h 2 FOFSE_HEAD_TIE=0 FOFSE_HEAD_TIE=1
WORKLOAD=C3 bash tools/gpu/abn.sh s3h3 2 FOFSE_HEAD_TIE=0 FOFSE_HEAD_TIE=1
