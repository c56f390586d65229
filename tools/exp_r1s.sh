timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for e in 1 0; do SDB_ELL=$e timeout 300 python tools/config_bench.py C1 --reps 5 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('ell=$e', d['config'], 'ms', round(d['seconds']*1e3,3), 'step_us', round(d['step_us'],2), 'gnnz', round(d['gnnz_vec_s'],1))"; done
