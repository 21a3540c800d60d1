timeout 1200 python tools/parity_study_batch.py C4 256 9100 8:1e-5 > gpurun_out/s3c_c4.log 2>&1; echo c4 rc=$?; tail -1 gpurun_out/s3c_c4.log
timeout 1200 python tools/parity_study_batch.py C4 256 31337 8:1e-5 > gpurun_out/s3c_c4b.log 2>&1; echo c4b rc=$?; tail -1 gpurun_out/s3c_c4b.log
timeout 1200 python tools/parity_study_batch.py C5 10 500 16:1e-5 > gpurun_out/s3c_c5.log 2>&1; echo c5 rc=$?; tail -1 gpurun_out/s3c_c5.log
timeout 1200 python tools/parity_study_batch.py C2 32 700 8:1e-5 > gpurun_out/s3c_c2.log 2>&1; echo c2 rc=$?; tail -1 gpurun_out/s3c_c2.log
timeout 1200 python tools/parity_study_batch.py C3 4 300 4:1e-5 > gpurun_out/s3c_c3.log 2>&1; echo c3 rc=$?; tail -1 gpurun_out/s3c_c3.log
