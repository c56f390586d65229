# C2: probe batch (L2-resident recurrence blocks) x store hint (.cs vs default write-back)
cp paper_1308_5467_b200/libspecdens_b200.so /tmp/main.so
for lib in main wb; do
  if [ $lib = wb ]; then cp exp_lib/lib_wb.so paper_1308_5467_b200/libspecdens_b200.so; fi
  for b in 64 32 16 8; do SDB_BATCH=$b timeout 300 python tools/config_bench.py C2 --reps 5 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$lib batch=$b', 'ms', round(d['seconds']*1e3,3), 'step_us', round(d['step_us'],2), 'gnnz', round(d['gnnz_vec_s'],1))"; done
  timeout 300 python tools/config_bench.py C5 --reps 1 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('$lib C5 s', round(d['seconds'],4), 'gnnz', round(d['gnnz_vec_s'],1))"
done
cp /tmp/main.so paper_1308_5467_b200/libspecdens_b200.so
