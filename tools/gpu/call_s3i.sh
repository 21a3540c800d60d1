timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s3i_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/s3i_tests.log
for t in 1e-9 1e-11 1e-12; do FOFSE_HEAD_TIE_TAU=$t timeout 900 python tools/parity_study_batch.py C3 4 300 4:1e-5 2>&1 | grep C3 | sed "s/^/tau=$t /"; done
FOFSE_HEAD_TIE_TAU=1e-11 timeout 900 python tools/parity_study_batch.py C4 64 2207 8:1e-5 2>&1 | grep C4
bash tools/gpu/abn.sh s3i 1 FOFSE_HEAD_TIE=0 FOFSE_HEAD_TIE_TAU=1e-9 FOFSE_HEAD_TIE_TAU=1e-11 FOFSE_HEAD_TIE_TAU=1e-12
WORKLOAD=C3 bash tools/gpu/abn.sh s3i3 1 FOFSE_HEAD_TIE=0 FOFSE_HEAD_TIE_TAU=1e-9 FOFSE_HEAD_TIE_TAU=1e-11 FOFSE_HEAD_TIE_TAU=1e-12
