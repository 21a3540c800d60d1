timeout 1500 python tools/stress_gpu.py 150 311 > gpurun_out/s3r_stress1.log 2>&1; echo s1 rc=$?; tail -1 gpurun_out/s3r_stress1.log
timeout 1500 python tools/stress_gpu2.py 150 313 > gpurun_out/s3r_stress2.log 2>&1; echo s2 rc=$?; tail -1 gpurun_out/s3r_stress2.log
