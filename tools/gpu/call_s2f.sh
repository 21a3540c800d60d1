set -x
FOFSE_V2R_VAR=6 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s2f_tests6.log 2>&1; echo tests6 rc=$?
tail -2 gpurun_out/s2f_tests6.log
bash tools/gpu/abn.sh s2f 2 FOFSE_V2R_VAR=0 FOFSE_V2R_VAR=6 FOFSE_V2R_VAR=7 FOFSE_V2R_VAR=8
