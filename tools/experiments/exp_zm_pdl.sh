# C2 z-march segment count / persistent grid re-swept with PDL-chained steps
for nzs in 0 3 4 5 6 8; do
  SDB_ZM_NZS=$nzs timeout 300 python tools/config_bench.py C2 --reps 5 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('nzs=$nzs', round(d['seconds']*1e3,3), 'ms', round(d['step_us'],2), 'us/step')"
done
for g in 148 296 444; do
  SDB_ZM_GRID=$g timeout 300 python tools/config_bench.py C2 --reps 5 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('grid=$g', round(d['seconds']*1e3,3), 'ms', round(d['step_us'],2), 'us/step')"
done
