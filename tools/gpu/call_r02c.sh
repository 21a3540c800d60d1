set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || true
timeout 600 python -m pytest tests/test_gpu_exact.py tests/test_ref_link.py -q > gpurun_out/pytest_exact.log 2>&1; echo "exact rc=$?"
tail -n 30 gpurun_out/pytest_exact.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -n 5 gpurun_out/pytest_gpu.log
mkdir -p gpurun_out/san
for gw in 1 2; do
  FOFSE_V2_REAL_GW=$gw timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_case.py > gpurun_out/san/racecheck_gw$gw.log 2>&1; echo "racecheck gw$gw rc=$?"
  tail -n 4 gpurun_out/san/racecheck_gw$gw.log
done
timeout 1200 compute-sanitizer --tool synccheck python tools/sanitize_case.py > gpurun_out/san/synccheck.log 2>&1; echo "synccheck rc=$?"; tail -n 4 gpurun_out/san/synccheck.log
timeout 1200 compute-sanitizer --tool memcheck python tools/sanitize_case.py > gpurun_out/san/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -n 4 gpurun_out/san/memcheck.log
