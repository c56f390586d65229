set -x
timeout 300 python -m pytest tests/test_gpu_zmarch.py -x -q > gpurun_out/zm_pytest.log 2>&1; echo EXIT $? >> gpurun_out/zm_pytest.log
tail -30 gpurun_out/zm_pytest.log
if grep -q "passed" gpurun_out/zm_pytest.log && ! grep -q "failed" gpurun_out/zm_pytest.log; then
for c in ${ZM_CFGS:-0 1 2 3 4 6}; do echo "cfg $c"; SDB_ZM_CFG=$c timeout 300 python tools/config_bench.py C2 C5 --reps 3 2>&1 | grep -v Warn; done > gpurun_out/zm_sweep.log 2>&1
fi
