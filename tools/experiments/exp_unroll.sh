# C4 variants (exp_lib/lib_<v>.so vs main), interleaved: unroll sweeps, lz_update_proj min-blocks (m2)
cp paper_1308_5467_b200/libspecdens_b200.so /tmp/main.so
for v in main w4 w16 main w4 w16 main; do
  if [ $v = main ]; then cp /tmp/main.so paper_1308_5467_b200/libspecdens_b200.so; else cp exp_lib/lib_$v.so paper_1308_5467_b200/libspecdens_b200.so; fi
  timeout 300 python tools/config_bench.py C4 --reps 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', round(d['seconds'],4), round(d['frac_vs_minimal_bytes'],3))"
done
cp /tmp/main.so paper_1308_5467_b200/libspecdens_b200.so
