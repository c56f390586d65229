# ncu capture of the fused step kernel on one config.  usage: bash tools/profile_config.sh <tag> <config> [extra args]
tag=$1; cfg=$2; shift 2
python tools/config_bench.py $cfg --reps 1 "$@" > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"cheb_step" -s 3 -c 1 -o gpurun_out/prof_$tag \
    python tools/config_bench.py $cfg --reps 1 "$@" > gpurun_out/ncu_$tag.log 2>&1
echo "profile $tag rc=$?"
