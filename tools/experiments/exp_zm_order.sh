# z-march item order: raster (0) against wave groups of compact strips (1), with z segment counts and strip widths
run() {
  echo "$*"
  env "$@" timeout 300 python tools/config_bench.py C2 C5 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print('   ', d['config'], round(d['step_us'], 1), 'us/step', round(d['frac_of_peak'], 3))
"
}
for rep in 1 2; do
run SDB_ZM_ORDER=0
run SDB_ZM_ORDER=1 SDB_ZM_SW=8
done
run SDB_ZM_ORDER=1 SDB_ZM_SW=4
run SDB_ZM_ORDER=1 SDB_ZM_SW=16
run SDB_ZM_ORDER=0 SDB_ZM_NZS=4
run SDB_ZM_ORDER=1 SDB_ZM_SW=8 SDB_ZM_NZS=4
run SDB_ZM_ORDER=1 SDB_ZM_SW=8 SDB_ZM_NZS=8
run SDB_ZM_ORDER=1 SDB_ZM_SW=8 SDB_ZM_NZS=16
for o in 0 1; do
  SDB_ZM_ORDER=$o ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:cheb_step_zmarch -s 3 -c 1 python tools/prof_step.py C5 12 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/  order=$o /"
done
# re-check of the L2 hint default on this box (C5 varies by ~2 % between boxes)
for rep in 1 2 3; do
run SDB_ZM_HINT=0
run SDB_ZM_HINT=2
done
