# z-march tile configuration / ring depth sweep on C2 and C5 (after the shared 4x3 window change)
for cfg in 3 0 2 1 4; do
  for r in 8 6; do
    echo "SDB_ZM_CFG=$cfg SDB_ZM_R=$r"
    SDB_ZM_CFG=$cfg SDB_ZM_R=$r timeout 300 python tools/config_bench.py C2 C5 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print('   ', d['config'], round(d['step_us'], 1), 'us/step', round(d['frac_of_peak'], 3))
"
  done
done
