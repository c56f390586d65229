timeout 900 python -m pytest tests/test_gpu_rowpart.py tests/test_gpu_distributed.py -x -q > gpurun_out/pytest_rp.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_rp.log
timeout 600 python tools/rowpart_bench.py --n 128 --slabs 2 --degree 200
timeout 600 python tools/rowpart_bench.py --n 256 --slabs 2 --degree 100
