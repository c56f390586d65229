set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" 
for v in "SDB_BAND_S=16" "SDB_BAND_S=8" "SDB_BAND=0"; do
env $v timeout 900 python tools/config_bench.py C3 --reps 2 2>&1 | tail -1 | cut -c1-400 | sed "s/^/$v /" | tee -a gpurun_out/r2b_c3.txt
done
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 | tee gpurun_out/r2b_pytest.txt
