set -x
timeout 900 python bench.py > gpurun_out/final2_c4.json 2>gpurun_out/final2_c4.err; echo c4 rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final2_ref.json 2>/dev/null; echo ref rc=$?
for w in C1 C2 C3 C5; do timeout 600 python bench.py --workload $w --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/final2_$w.json 2>/dev/null; echo $w rc=$?; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_C4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu1 rc=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k2v2r_kernel --launch-skip 2 -c 1 -o gpurun_out/r02_prof_k2v2r python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu2 rc=$?
