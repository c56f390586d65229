python -m pytest tests/test_gpu_band.py -x -q 2>&1 | tail -2
for v in "SDB_BAND_DIAG=0" "SDB_BAND_S=8"; do
env $v timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum \
  --clock-control none -k regex:cheb_step_band -s 3 -c 1 python tools/prof_step.py C3 12 2>&1 | grep -E "duration|dram__|hit_rate|inst_exec" | sed "s/^/$v /"
done
timeout 600 python tools/config_bench.py C3 --reps 2 2>&1 | tail -1 | cut -c1-300
