# sweep prebuilt library variants (tools/variants/lib_v*.so) on the C2 bench
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
cp paper_1308_5467_b200/libspecdens_b200.so /tmp/lib_orig.so
run() { # tag env...
  tag=$1; shift
  env "$@" python bench.py --steps 10 --warmup 3 --no-cpu-baseline $BARGS > gpurun_out/v_$tag.json 2>gpurun_out/v_err.log || tail -3 gpurun_out/v_err.log
  python -c "import json;d=json.load(open('gpurun_out/v_$tag.json'));print('$tag', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'us', round(d['roofline']['avg_launch_us'],1))"
}
for v in $VARIANTS; do
  cp tools/variants/lib_v$v.so paper_1308_5467_b200/libspecdens_b200.so
  for fmt in csr stencil; do
    BARGS="--format $fmt"
    run v${v}_${fmt}_L32 X=1
    run v${v}_${fmt}_L16 SDB_LANES=16
  done
done
cp /tmp/lib_orig.so paper_1308_5467_b200/libspecdens_b200.so
