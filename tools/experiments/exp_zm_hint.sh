# z-march: L2 cache policies on the TMA loads (SDB_ZM_HINT: 1 = w_{k-1}/v0 boxes evict_first, 2 = x boxes evict_last)
for rep in 1 2; do
for h in 0 1 2 3; do
  echo "SDB_ZM_HINT=$h"
  SDB_ZM_HINT=$h timeout 300 python tools/config_bench.py C2 C5 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print('   ', d['config'], round(d['step_us'], 1), 'us/step', round(d['frac_of_peak'], 3))
"
done
done
# DRAM bytes of one C5 step under each policy
for h in 0 1 3; do
  SDB_ZM_HINT=$h ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none \
    -k regex:cheb_step_zmarch -s 3 -c 1 python tools/prof_step.py C5 12 2>&1 | grep -E "dram__|gpu__time|lts__t" | sed "s/^/  hint=$h /"
done
