# fused-pair sweep: per-step kernel time for C2 / C5 (config_bench: step_us = kernel time / steps)
for c in ${ZM_CFGS:-3 0 2}; do echo "fused cfg $c"; SDB_ZM_CFG=$c timeout 300 python tools/config_bench.py C2 C5 --reps 3 2>&1 | grep -o '"config": "C.\|"step_us": [0-9.]*' | paste - -; done
echo "single-step cfg 3"; SDB_ZM_FUSE=0 SDB_ZM_CFG=3 timeout 300 python tools/config_bench.py C2 C5 --reps 3 2>&1 | grep -o '"config": "C.\|"step_us": [0-9.]*' | paste - -
timeout 300 python bench.py > gpurun_out/bench_fused.json 2>gpurun_out/bench_fused.err; tail -c 1500 gpurun_out/bench_fused.json
