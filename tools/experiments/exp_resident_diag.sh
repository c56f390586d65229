# C1 resident kernel under its timing diagnostics (wrong results for diag != 0)
for d in 0 1 2 4 6; do
  echo "SDB_RES_DIAG=$d"
  SDB_RES_DIAG=$d timeout 300 python tools/config_bench.py C1 --reps 20 2>&1 | tail -1 | grep -o "\"seconds\": [0-9.e-]*\|\"step_us\": [0-9.]*" | paste - -
done
