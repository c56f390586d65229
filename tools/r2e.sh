mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_band.py -x -q 2>&1 | tail -5
timeout 600 python tools/band_diag.py 100 "" SDB_BAND_DIAG=12 2>&1 | tail -4 | tee gpurun_out/r2e_diag.txt
