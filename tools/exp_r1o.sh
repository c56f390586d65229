timeout 900 python -m pytest tests/test_gpu_zmarch.py tests/test_gpu_rowpart.py -x -q > gpurun_out/pytest_zm.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_zm.log
for w in 0 4 8 16; do SDB_ZM_SWZ=$w timeout 300 python tools/config_bench.py C2 C5 --reps 3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('swz=$w', d['config'], round(d['step_us'],2), round(d['frac_of_peak'],3))"; done
