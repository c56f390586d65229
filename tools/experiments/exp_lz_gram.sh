# C4 Lanczos: two-pass Gram-corrected reorthogonalisation against the three-pass schedule
for rep in 1 2; do
for g in 0 1; do
  echo "SDB_LZ_GRAM=$g"
  SDB_LZ_GRAM=$g timeout 600 python tools/config_bench.py C4 2>&1 | tail -1
done
done
