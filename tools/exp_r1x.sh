for c in 3 7 8; do SDB_ZM_CFG=$c timeout 300 python tools/config_bench.py C2 C5 --reps 3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('cfg=$c', d['config'], round(d['step_us'],2), round(d['frac_of_peak'],3))"; done
