timeout 900 python -m pytest tests/test_gpu_rowpart.py tests/test_gpu_distributed.py tests/test_native_abi.py -x -q > gpurun_out/pytest_rp.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_rp.log
timeout 600 python tools/rowpart_bench.py --n 256 --slabs 2 --degree 100
timeout 600 python tools/rowpart_bench.py --n 256 --slabs 8 --degree 60
