set -x
timeout 900 python bench.py --impl reference > gpurun_out/s2p_ref.json 2>gpurun_out/s2p_ref.err; echo ref rc=$?
tail -c 600 gpurun_out/s2p_ref.json
