set -x
timeout 900 python -m pytest tests/test_gpu_k1p.py -x -q > gpurun_out/s2g_k1p.log 2>&1; echo k1ptest rc=$?
tail -15 gpurun_out/s2g_k1p.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s2g_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/s2g_tests.log
bash tools/gpu/abn.sh s2g 3 FOFSE_K1P=0 FOFSE_K1P=1
