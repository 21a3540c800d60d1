set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/k1h_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/k1h_tests.log
bash tools/gpu/abn.sh k1h3 2 FOFSE_K1H=0 FOFSE_K1H=1
