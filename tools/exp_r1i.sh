timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python tools/rowpart_bench.py --n 256 --slabs 2 --degree 100
timeout 600 python tools/rowpart_bench.py --n 256 --slabs 8 --degree 60
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2>gpurun_out/bench_err.log; python -c "import json;d=json.load(open('gpurun_out/bench_c2.json'));print('C2', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'us', round(d['roofline']['avg_launch_us'],1), 'e2e', round(d['e2e']['value'],1), d['clocks'])"
timeout 300 python tools/config_bench.py C5 --reps 2 2>&1 | tail -1 | cut -c1-300
