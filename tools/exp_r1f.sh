timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python tools/config_bench.py C4 --reps 1 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c4.csv python tools/config_bench.py C4 --reps 1 > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches_c4.csv gpurun_out/launch_summary_c4.txt "C4 Lanczos (m=100, 128 probes), ncu launch list" | head -20
