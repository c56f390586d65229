for r in 6 7 8 10 12; do SDB_ZM_R=$r timeout 300 python tools/config_bench.py C2 C5 --reps 3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('R=$r', d['config'], round(d['step_us'],2), round(d['frac_of_peak'],3))"; done
