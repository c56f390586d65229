# correctness + C2 bench in csr and stencil form
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for fmt in csr stencil; do
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --format $fmt > gpurun_out/bench_$fmt.json 2>gpurun_out/bench_err.log || tail -5 gpurun_out/bench_err.log
  python -c "import json;d=json.load(open('gpurun_out/bench_$fmt.json'));print('$fmt', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'us', round(d['roofline']['avg_launch_us'],1), 'e2e', round(d['e2e']['value'],1), d['clocks'])"
done
