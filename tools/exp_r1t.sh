timeout 900 python -m pytest tests/test_gpu_lanczos.py tests/test_gpu_haydock.py tests/test_gpu_interval.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_lz.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_lz.log
for f in 1 0; do SDB_LZ_TMA=$f timeout 300 python tools/config_bench.py C4 --reps 3 2>&1 | tail -1 | cut -c1-250 | sed "s/^/tma=$f /"; done
