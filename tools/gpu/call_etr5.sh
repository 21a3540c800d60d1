set -x
timeout 1500 python -m pytest tests -m gpu -x -q -k "parity or guard or frame" > gpurun_out/etr5_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/etr5_tests.log
timeout 900 python bench.py --no-cpu-baseline --no-fp64 --steps 3 --warmup 3 > gpurun_out/etr5.json 2>/dev/null; echo c4 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/etr5.json').read().strip().splitlines()[-1]); print('C4', round(d['value']), round(d['e2e']['value']), d['parity']['max_px'], d['parity']['blocks_over_0.5'], d['parity']['dpsnr_db'])"
bash tools/gpu/abn.sh etr5 2 FOFSE_ETR=0 FOFSE_ETR=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_etr5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-fp64 > /dev/null 2>&1; echo ncu rc=$?
