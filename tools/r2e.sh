mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_gpu_band.py -x -q 2>&1 | tail -12
timeout 300 python tools/band_diag.py 100 "" SDB_BAND_NB=3 SDB_BAND_NB=10 SDB_BAND_DIAG=12 2>&1 | tail -8 | tee gpurun_out/r2e_diag.txt
