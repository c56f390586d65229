# C4: lz_update streamed by basis vector (SDB_LZ_UPD_STREAM=1) vs the row-group form (0), interleaved
timeout 600 python -m pytest tests/test_gpu_lanczos.py tests/test_gpu_haydock.py tests/test_gpu_interval.py tests/test_gpu_comparison.py -x -q 2>&1 | tail -2
for v in 1 0 1 0 1; do
  SDB_LZ_UPD_STREAM=$v timeout 300 python tools/config_bench.py C4 --reps 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('stream=$v', round(d['seconds'],4), round(d['frac_vs_minimal_bytes'],3))"
done
