python tools/prof_step.py C2 20 > gpurun_out/prof_c2.log 2>&1
SDB_ZM_CFG=3 timeout 600 ncu --set full --import-source on -k regex:cheb_step_zmarch --launch-skip 4 -c 1 -o gpurun_out/zm_c2 -f python tools/prof_step.py C2 20 > gpurun_out/ncu_zm_c2.log 2>&1
SDB_ZM_CFG=3 timeout 900 ncu --set full --import-source on -k regex:cheb_step_zmarch --launch-skip 4 -c 1 -o gpurun_out/zm_c5 -f python tools/prof_step.py C5 12 > gpurun_out/ncu_zm_c5.log 2>&1
tail -3 gpurun_out/ncu_zm_c2.log gpurun_out/ncu_zm_c5.log
