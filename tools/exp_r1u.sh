timeout 600 python -m pytest tests/test_gpu_lanczos.py -x -q 2>&1 | tail -1
for r in 0 1 2 4; do SDB_LZ_PROJ_ROWS=$r timeout 300 python tools/config_bench.py C4 --reps 3 2>&1 | tail -1 | cut -c1-200 | sed "s/^/rows=$r /"; done
