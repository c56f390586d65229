# Programmatic dependent launch between recurrence steps: on (default) vs SDB_PDL=0
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pdl_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pdl_tests.log
for pdl in 0 1; do
  SDB_PDL=$pdl timeout 600 python tools/config_bench.py C1 C2 C3 C5 --reps 3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('pdl=$pdl', d['config'], 'ms', round(d['seconds']*1e3,3), 'step_us', round(d.get('step_us',0),2), 'gnnz', round(d['gnnz_vec_s'],1))"
done
SDB_PDL=0 python bench.py --no-cpu-baseline > gpurun_out/bench_pdl0.json 2>&1; tail -1 gpurun_out/bench_pdl0.json | cut -c1-200
python bench.py --no-cpu-baseline > gpurun_out/bench_pdl1.json 2>&1; tail -1 gpurun_out/bench_pdl1.json | cut -c1-200
