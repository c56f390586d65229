set -x
python -m pytest tests/test_gpu_band.py -x -q 2>&1 | tail -5
SDB_BAND_S=8 python -m pytest tests/test_gpu_band.py -x -q 2>&1 | tail -5
timeout 600 python tools/config_bench.py C3 --reps 2 2>&1 | tail -1
SDB_BAND_S=8 timeout 600 python tools/config_bench.py C3 --reps 2 2>&1 | tail -1
