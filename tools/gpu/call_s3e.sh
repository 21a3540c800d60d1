timeout 900 python tools/parity_study_batch.py C3 4 300 5:1e-5 6:1e-5 8:1e-5 2>&1 | grep C3
timeout 900 python tools/parity_study_batch.py C3 4 900 4:1e-5 6:1e-5 8:1e-5 2>&1 | grep C3
