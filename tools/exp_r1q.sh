# duplicate-store removal (main) and default-caching variant vs probe batch on C2 / C5
for b in 64 16 8; do SDB_BATCH=$b timeout 300 python tools/config_bench.py C2 --reps 5 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('main batch=$b', d['config'], 'ms', round(d['seconds']*1e3,3), 'step_us', round(d['step_us'],2))"; done
timeout 300 python tools/config_bench.py C5 --reps 2 2>&1 | tail -1 | cut -c1-200
cp paper_1308_5467_b200/libspecdens_b200.so /tmp/main.so
cp exp_lib/lib_nocs.so paper_1308_5467_b200/libspecdens_b200.so
for b in 64 16 8; do SDB_BATCH=$b timeout 300 python tools/config_bench.py C2 --reps 5 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('nocs batch=$b', d['config'], 'ms', round(d['seconds']*1e3,3), 'step_us', round(d['step_us'],2))"; done
cp /tmp/main.so paper_1308_5467_b200/libspecdens_b200.so
