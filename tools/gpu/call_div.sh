set -x
python tools/divergence_study.py C4 64 2207 4 gpurun_out/div_c4_h4.npz > gpurun_out/div_c4_h4.log 2>&1
python tools/divergence_study.py C4 64 2207 8 gpurun_out/div_c4_h8.npz > gpurun_out/div_c4_h8.log 2>&1
python tools/divergence_study.py C5 4 500 4 gpurun_out/div_c5_h4.npz > gpurun_out/div_c5_h4.log 2>&1
python tools/divergence_study.py C5 4 500 8 gpurun_out/div_c5_h8.npz > gpurun_out/div_c5_h8.log 2>&1
python tools/divergence_study.py C5 4 500 16 gpurun_out/div_c5_h16.npz > gpurun_out/div_c5_h16.log 2>&1
python tools/divergence_study.py C2 8 700 4 gpurun_out/div_c2_h4.npz > gpurun_out/div_c2_h4.log 2>&1
python tools/divergence_study.py C3 1 300 4 gpurun_out/div_c3_h4.npz > gpurun_out/div_c3_h4.log 2>&1
tail -n 3 gpurun_out/div_*.log
