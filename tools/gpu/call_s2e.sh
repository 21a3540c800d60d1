set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s2e_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/s2e_tests.log
bash tools/gpu/abn.sh s2e 3 FOFSE_HEAD_NARROW=0 FOFSE_HEAD_NARROW=1
