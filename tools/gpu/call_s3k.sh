timeout 600 python -m pytest tests/test_gpu_parity.py -k "exact_ties or default_on" -q > gpurun_out/s3k_t.log 2>&1; echo t rc=$?; tail -2 gpurun_out/s3k_t.log
timeout 1200 python tools/parity_study_batch.py C4 256 2207 8:1e-5 2>&1 | grep C4
timeout 1200 python tools/parity_study_batch.py C4 256 9100 8:1e-5 2>&1 | grep C4
timeout 1200 python tools/parity_study_batch.py C4 256 31337 8:1e-5 2>&1 | grep C4
timeout 1200 python tools/parity_study_batch.py C5 10 500 16:1e-5 2>&1 | grep C5
timeout 1200 python tools/parity_study_batch.py C2 32 700 8:1e-5 2>&1 | grep C2
timeout 1200 python tools/parity_study_batch.py C3 4 300 4:1e-5 2>&1 | grep C3
timeout 1200 python tools/parity_study_batch.py C3 4 900 4:1e-5 2>&1 | grep C3
