set -e
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1 || { echo PYTEST_FAIL; tail -30 gpurun_out/pytest_gpu.log; }
tail -2 gpurun_out/pytest_gpu.log
for fmt in csr stencil; do for P in 0 16 32 64 128 256 448; do
  SDB_PANEL_ROWS=$P python bench.py --steps 10 --warmup 3 --no-cpu-baseline --format $fmt > gpurun_out/sweep_${fmt}_$P.json 2>gpurun_out/sweep_err.log || tail -5 gpurun_out/sweep_err.log
  python -c "import json;d=json.load(open('gpurun_out/sweep_${fmt}_$P.json'));print('$fmt P=$P', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'us', round(d['roofline']['avg_launch_us'],1), 'e2e', round(d['e2e']['value'],1))"
done; done
