# Final round evidence: GPU suite, smoke, bench lines (C2 headline + reference arm + C5), launch lists,
# ncu of the C2 step, per-config timings (C1-C5), C4 launch list.
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 bash tools/round_evidence.sh
timeout 600 python bench.py --config C5 --format stencil --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2>&1; echo "c5 rc=$?"
timeout 900 python tools/config_bench.py C1 C2 C3 C4 C5 --reps 3 > gpurun_out/configs.jsonl 2>&1; echo "cfg rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c4.csv \
    python tools/config_bench.py C4 --reps 1 > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
tail -1 gpurun_out/bench_default.json
