# probe-batch size on C2: does a batch whose recurrence blocks fit L2 run from L2?
for b in 64 32 16 8; do SDB_BATCH=$b timeout 300 python tools/config_bench.py C2 --reps 5 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('batch=$b', d['config'], 'seconds', round(d['seconds']*1e3,3), 'ms', 'step_us', round(d['step_us'],2), 'gnnz', round(d['gnnz_vec_s'],1))"; done
