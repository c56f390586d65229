# One gpurun payload: the round's measured evidence into gpurun_out/<tag>_* (copied to profiles/ afterwards).
#   gpurun --timeout 3400 -- 'bash tools/round_evidence.sh r02'
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/${TAG}_box.txt
lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" >> $O/${TAG}_box.txt
# bench lines (the driver's command, then the other KPM configs) and the reference arm
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${TAG}_bench_c3.json 2> $O/${TAG}_bench_c3.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/${TAG}_bench_reference_c3.json 2>> $O/${TAG}_bench_c3.err
python bench.py --config C2 --steps 20 --warmup 5 > $O/${TAG}_bench_c2.json 2>> $O/${TAG}_bench_c3.err
python bench.py --config C5 --steps 3 --warmup 3 > $O/${TAG}_bench_c5.json 2>> $O/${TAG}_bench_c3.err
python bench.py --config C1 --steps 50 --warmup 10 > $O/${TAG}_bench_c1.json 2>> $O/${TAG}_bench_c3.err
# every config with its CPU baseline beside it
python tools/config_bench.py C1 C2 C3 C4 C5 --cpu > $O/${TAG}_configs.jsonl 2> $O/${TAG}_configs.err
# launch list of the bench command (after it exited 0 without ncu, above)
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $O/${TAG}_launches_c3.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cold > $O/${TAG}_ncu_launch.log 2>&1
python tools/launch_summary.py $O/${TAG}_launches_c3.csv $O/${TAG}_launches_c3.txt \
  "ncu launch list: python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cold (C3)" > /dev/null
# C4 Lanczos launch list (two-pass Gram-corrected reorthogonalisation)
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/${TAG}_launches_c4.csv \
  python tools/config_bench.py C4 --reps 1 > $O/${TAG}_ncu_launch_c4.log 2>&1
python tools/launch_summary.py $O/${TAG}_launches_c4.csv $O/${TAG}_launches_c4.txt \
  "C4 Lanczos (m=100, 128 probes) launch list, config_bench --reps 1" > /dev/null
# ncu --set full of one band step and one C5 z-march step
ncu --set full --import-source on --clock-control none -k regex:cheb_step_band -s 3 -c 1 -o $O/${TAG}_band_c3 -f \
  python tools/prof_step.py C3 12 > $O/${TAG}_ncu_band.log 2>&1
python tools/ncu_summary.py $O/${TAG}_band_c3.ncu-rep 25 > $O/${TAG}_ncu_band_c3.txt 2>&1
ncu --set full --clock-control none -k regex:cheb_step_zmarch -s 3 -c 1 -o $O/${TAG}_zmarch_c5 -f \
  python tools/prof_step.py C5 12 > $O/${TAG}_ncu_zm5.log 2>&1
python tools/ncu_summary.py $O/${TAG}_zmarch_c5.ncu-rep > $O/${TAG}_ncu_zmarch_c5.txt 2>&1
# the reference's own test modules against the drop-in
python -m pytest tests/test_reference_suite.py -m gpu -q -rA 2>&1 | tail -15 > $O/${TAG}_reference_suite.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.txt 2>&1
ls -la $O | tail -30
