# C1: cluster-resident recurrence (one launch) against PDL-chained per-step launches
for rep in 1 2 3; do
for r in 0 1; do
  echo "SDB_RESIDENT=$r"
  SDB_RESIDENT=$r timeout 300 python tools/config_bench.py C1 --reps 20 2>&1 | tail -1 | cut -c1-330
done
done
