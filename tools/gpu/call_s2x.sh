timeout 900 python -m pytest tests/test_gpu_k1p.py -x -q > gpurun_out/s2x.log 2>&1; echo rc=$?; tail -15 gpurun_out/s2x.log
