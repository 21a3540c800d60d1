set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/etr6_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/etr6_tests.log
