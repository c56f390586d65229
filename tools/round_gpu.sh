# GPU tests + round evidence + C5 profile, one call.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 bash tools/round_evidence.sh
timeout 600 bash tools/profile_step.sh c5 --config C5 --format stencil --steps 1
tail -1 gpurun_out/bench_default.json
