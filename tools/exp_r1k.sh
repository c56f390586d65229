timeout 900 python -m pytest tests/test_gpu_lanczos.py tests/test_gpu_haydock.py tests/test_gpu_interval.py -x -q > gpurun_out/pytest_lz.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_lz.log
for f in 1 0; do SDB_LZ_FUSED=$f timeout 300 python tools/config_bench.py C4 --reps 2 2>&1 | tail -1 | cut -c1-330 | sed "s/^/fused=$f /"; done
