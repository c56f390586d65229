# one gpurun payload: GPU tests (all, or those given as arguments), log under gpurun_out/
mkdir -p gpurun_out
timeout 3000 python -m pytest ${@:-tests} -m gpu -q 2>&1 | tail -150 > gpurun_out/gpu_suite.txt
tail -5 gpurun_out/gpu_suite.txt
