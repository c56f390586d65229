set -x
mkdir -p gpurun_out
python tools/band_diag.py 100 2>&1 | tee gpurun_out/r2c_diag.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cheb_step_band -s 3 -c 1 -o gpurun_out/r2c_band_s16 -f python tools/prof_step.py C3 12 > gpurun_out/r2c_ncu.log 2>&1
tail -3 gpurun_out/r2c_ncu.log
