timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python tools/config_bench.py C2 C5 --reps 5 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], round(d['step_us'],2), round(d['frac_of_peak'],3), round(d['seconds'],4))"
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2>gpurun_out/bench_err.log; python -c "import json;d=json.load(open('gpurun_out/bench_c2.json'));print('C2 bench', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'us', round(d['roofline']['avg_launch_us'],1), 'e2e', round(d['e2e']['value'],1), d['clocks'])"
