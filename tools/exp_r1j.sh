# ncu of the three CGS kernels at a late Lanczos step (C4)
ncu --set full --clock-control none --import-source on -k regex:"lz_proj|lz_update" -s 270 -c 4 -o gpurun_out/prof_lz python tools/config_bench.py C4 --reps 1 > gpurun_out/ncu_lz.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/prof_lz.ncu-rep > gpurun_out/ncu_lz_summary.txt 2>&1; head -90 gpurun_out/ncu_lz_summary.txt
