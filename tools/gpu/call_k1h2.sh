bash tools/gpu/abn.sh k1h2 2 FOFSE_K1H=0 FOFSE_K1H=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_k1h.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu rc=$?
