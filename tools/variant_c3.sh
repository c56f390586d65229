cp paper_1308_5467_b200/libspecdens_b200.so /tmp/lib_orig.so
for v in 0 1 2 3 4; do
  cp tools/variants/lib_v$v.so paper_1308_5467_b200/libspecdens_b200.so
  python tools/config_bench.py C3 --reps 2 2>/dev/null | python -c "import sys,json; [print(\"v$v\", d[\"config\"], round(d[\"step_us\"],1), round(d[\"frac_of_peak\"],3), round(d[\"seconds\"],3)) for d in map(json.loads, sys.stdin)]"
done
cp /tmp/lib_orig.so paper_1308_5467_b200/libspecdens_b200.so
