for c in ${ZM_CFGS:-3 7 8 6}; do echo "cfg $c"; SDB_ZM_CFG=$c timeout 300 python tools/config_bench.py C2 C5 --reps 3 2>&1 | grep -o '"config": "C.\|"step_us": [0-9.]*' | paste - -; done
