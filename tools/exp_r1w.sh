timeout 600 python -m pytest tests/test_gpu_kpm.py -x -q 2>&1 | tail -1
timeout 300 python tools/config_bench.py C3 C1 --reps 2 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('far', d['config'], 'ms', round(d['seconds']*1e3,2), 'step_us', round(d['step_us'],2), 'gnnz', round(d['gnnz_vec_s'],1))"
timeout 300 python tools/config_bench.py C2 --format csr-raw --reps 3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('far', d['config'], d['format'], 'step_us', round(d['step_us'],2))"
