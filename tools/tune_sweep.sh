python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
run() { # tag env...
  tag=$1; shift
  env "$@" python bench.py --steps 10 --warmup 3 --no-cpu-baseline $BARGS > gpurun_out/t_$tag.json 2>gpurun_out/t_err.log || tail -3 gpurun_out/t_err.log
  python -c "import json;d=json.load(open('gpurun_out/t_$tag.json'));print('$tag', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'us', round(d['roofline']['avg_launch_us'],1), 'e2e', round(d['e2e']['value'],1))"
}
for fmt in csr stencil; do
  BARGS="--format $fmt"
  run ${fmt}_default X=1
  run ${fmt}_L16 SDB_LANES=16
  run ${fmt}_B4 SDB_BLOCKS_PER_SM=4
  run ${fmt}_P32 SDB_PANEL_ROWS=32
  run ${fmt}_P128 SDB_PANEL_ROWS=128
done
BARGS="--format stencil"; run stencil_generic SDB_STENCIL_GENERIC=1
