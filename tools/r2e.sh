mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_band.py -x -q 2>&1 | tail -5
timeout 600 python tools/band_diag.py 100 "" SDB_BAND_NB=2 SDB_BAND_DIAG=4 SDB_BAND_DIAG=12 SDB_BAND_DIAG=16 2>&1 | tail -8 | tee gpurun_out/r2e_diag.txt
