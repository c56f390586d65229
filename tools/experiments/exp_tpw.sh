# C4: first CGS projection with TPW basis vectors per warp (w read once per TPW); repeated, interleaved
for t in 2 0 4 0 2 0; do
  SDB_LZ_TPW=$t timeout 300 python tools/config_bench.py C4 --reps 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('tpw=$t', round(d['seconds'],4), round(d['frac_vs_minimal_bytes'],3))"
done
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
