mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multidevice.py tests/test_gpu_distributed.py -x -q 2>&1 | tail -25
