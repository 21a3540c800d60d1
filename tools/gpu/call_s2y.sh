timeout 1500 python tools/stress_gpu.py 150 211 > gpurun_out/s2y_stress1.log 2>&1; echo s1 rc=$?; tail -2 gpurun_out/s2y_stress1.log
timeout 1500 python tools/stress_gpu2.py 150 213 > gpurun_out/s2y_stress2.log 2>&1; echo s2 rc=$?; tail -2 gpurun_out/s2y_stress2.log
