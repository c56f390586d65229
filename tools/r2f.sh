mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cheb_step_band -s 3 -c 1 -o gpurun_out/r2f_band -f python tools/prof_step.py C3 12 > gpurun_out/r2f_ncu.log 2>&1
tail -2 gpurun_out/r2f_ncu.log
