timeout 900 python -m pytest tests/test_gpu_kpm.py tests/test_gpu_lanczos.py -x -q > gpurun_out/pytest_e.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_e.log
for c in 1 0; do SDB_COOP=$c timeout 300 python tools/config_bench.py C1 --reps 5 2>&1 | tail -1 | cut -c1-260 | sed "s/^/coop=$c /"; done
