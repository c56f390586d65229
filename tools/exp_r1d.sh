timeout 600 python -m pytest tests/test_gpu_lanczos.py tests/test_gpu_haydock.py -x -q > gpurun_out/pytest_lz.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_lz.log
for cfg in "SDB_LZ_VARIANT=0" "SDB_LZ_VARIANT=1" "SDB_LZ_VARIANT=2" "SDB_LZ_VARIANT=3" "SDB_LZ_FUSED=0"; do env $cfg timeout 300 python tools/config_bench.py C4 --reps 2 2>&1 | tail -1 | cut -c1-150 | sed "s/^/$cfg /"; done
