set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/parity_study.py C4 256 2207 4:1e-5:0 4:1e-5:16 4:1e-5:32 4:1e-5:64 6:1e-5:0 8:1e-5:0 10:1e-5:0 4:5e-6:32 4:5e-6:64 6:1e-5:32 > gpurun_out/ps_c4_2207.log 2>&1
python tools/parity_study.py C4 256 9100 4:1e-5:0 4:1e-5:16 4:1e-5:32 4:1e-5:64 6:1e-5:0 8:1e-5:0 10:1e-5:0 4:5e-6:32 4:5e-6:64 6:1e-5:32 > gpurun_out/ps_c4_9100.log 2>&1
python tools/parity_study.py C5 6 500 4:1e-5:0 4:1e-5:32 4:1e-5:64 8:1e-5:0 4:5e-6:64 > gpurun_out/ps_c5.log 2>&1
python tools/parity_study.py C2 16 700 4:1e-5:0 4:1e-5:32 4:1e-5:64 8:1e-5:0 4:5e-6:64 > gpurun_out/ps_c2.log 2>&1
python tools/parity_study.py C3 2 300 4:1e-5:0 4:1e-5:32 4:1e-5:64 4:5e-6:64 > gpurun_out/ps_c3.log 2>&1
tail -n 12 gpurun_out/ps_*.log
